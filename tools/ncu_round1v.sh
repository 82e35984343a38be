# Round-1 (v, final build) evidence refresh: full capture of one C5 phase-3 launch, the
# launch list of the bench command, and the blocked pivot kernel.
set -x
NCU=/usr/local/cuda/bin/ncu
B32="python bench.py --steps 1 --warmup 1 --no-secondary --no-cpu"
$B32 > gpurun_out/plain_b32_v.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:packed_gemm -s 41 -c 1 -o gpurun_out/prof_fw32k_packed_3b_v $B32 > gpurun_out/ncu_b32full_v.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_fw32768_r1v.csv $B32 > gpurun_out/ncu_b32list_v.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:fw_pivot_blocked -s 5 -c 1 -o gpurun_out/prof_pivot_blocked_v python tools/perf_pivot.py 1024 > gpurun_out/ncu_pivot_v.log 2>&1
ls -la gpurun_out | tail -5
