set -x
NCU=/usr/local/cuda/bin/ncu
B32="python bench.py --steps 1 --warmup 1 --no-secondary --no-cpu"
$B32 > gpurun_out/plain_b32.log 2>&1 && $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:short, .int.128, .int.64" -s 200 -c 1 -o gpurun_out/prof_fw32k_phase3 $B32 > gpurun_out/ncu_b32full.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_fw32768_r1b.csv $B32 > gpurun_out/ncu_b32list.log 2>&1
P="python tools/profile_kernels.py"
$P warshall_bits --reps 1 > gpurun_out/pw.log 2>&1 && $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_warshall_bits_r1b.csv $P warshall_bits --reps 1 > /dev/null 2>&1
