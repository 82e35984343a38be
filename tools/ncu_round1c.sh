set -x
NCU=/usr/local/cuda/bin/ncu
B32="python bench.py --steps 1 --warmup 1 --no-secondary --no-cpu"
$B32 > gpurun_out/plain_b32.log 2>&1 && $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:short, .int.128, .int.64" -s 100 -c 1 -o gpurun_out/prof_fw32k_b256_phase3 $B32 > gpurun_out/ncu_b32full.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_fw32768_r1c.csv $B32 > gpurun_out/ncu_b32list.log 2>&1
