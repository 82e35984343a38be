set -x
NCU=/usr/local/cuda/bin/ncu
B8="python bench.py --n 8192 --steps 2 --warmup 1 --no-secondary --no-cpu"
$B8 > gpurun_out/plain_b8.log 2>&1 && $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fw8192.csv $B8 > gpurun_out/ncu_b8.log 2>&1
B32="python bench.py --steps 1 --warmup 1 --no-secondary --no-cpu"
$B32 > gpurun_out/plain_b32.log 2>&1 && $NCU --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_fw32768.csv $B32 > gpurun_out/ncu_b32.log 2>&1
P="python tools/profile_kernels.py"
$P gemm_u16 > gpurun_out/p1.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:semiring_gemm -s 1 -c 1 -o gpurun_out/prof_gemm_u16 $P gemm_u16 > gpurun_out/ncu_p1.log 2>&1
$P gemm_u8 > gpurun_out/p2.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:semiring_gemm -s 1 -c 1 -o gpurun_out/prof_gemm_u8 $P gemm_u8 > gpurun_out/ncu_p2.log 2>&1
$P tc > gpurun_out/p3.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:bool_i8 -s 1 -c 1 -o gpurun_out/prof_tc $P tc > gpurun_out/ncu_p3.log 2>&1
$P fw8k --reps 1 > gpurun_out/p4.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:semiring_gemm -s 21 -c 1 -o gpurun_out/prof_fw_phase3 $P fw8k --reps 1 > gpurun_out/ncu_p4.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_warshall_bits.csv $P warshall_bits --reps 1 > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_warshall_tc.csv $P warshall_tc --reps 1 > /dev/null 2>&1
ls -la gpurun_out/
