#!/bin/bash
# Parameterised ncu capture (replaces the per-run ncu_round1*.sh scripts).
# Always runs the command once WITHOUT ncu first; ncu only if that exits 0.
#
#   tools/ncu.sh full TAG KERNEL_REGEX SKIP COUNT -- cmd ...   # --set full capture -> gpurun_out/TAG.ncu-rep
#   tools/ncu.sh list TAG COUNT -- cmd ...                     # launch list -> gpurun_out/TAG.csv
#
# Per-launch times in a launch list are cold-cache and serialised (ncu), so
# compare shares of the step with the bench, not absolute times.
set -u
NCU=/usr/local/cuda/bin/ncu
mode=$1; tag=$2; shift 2
mkdir -p gpurun_out
if [ "$mode" = full ]; then
  regex=$1; skip=$2; count=$3; shift 3
else
  count=$1; shift 1
fi
[ "$1" = "--" ] && shift
"$@" > "gpurun_out/${tag}_plain.log" 2>&1 || { echo "plain run failed: $tag"; tail -20 "gpurun_out/${tag}_plain.log"; exit 1; }
if [ "$mode" = full ]; then
  $NCU --set full --clock-control none --import-source on -k "regex:$regex" -s "$skip" -c "$count" \
       -f -o "gpurun_out/$tag" "$@" > "gpurun_out/${tag}_ncu.log" 2>&1
else
  $NCU --metrics gpu__time_duration.sum --clock-control none -c "$count" --csv \
       --log-file "gpurun_out/$tag.csv" "$@" > "gpurun_out/${tag}_ncu.log" 2>&1
fi
echo "ncu $mode $tag rc=$?"
