set -x
NCU=/usr/local/cuda/bin/ncu
P="python tools/profile_kernels.py"
$P tc8k --reps 2 > gpurun_out/pj1.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:bool_i8_gemm -s 1 -c 1 -o gpurun_out/prof_tc8k $P tc8k --reps 2 > gpurun_out/ncu_pj1.log 2>&1
$P gemm_u16 --reps 2 > gpurun_out/pj2.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:packed_gemm -s 1 -c 1 -o gpurun_out/prof_c3u16_packed $P gemm_u16 --reps 2 > gpurun_out/ncu_pj2.log 2>&1
$P warshall_bits16k --reps 1 > gpurun_out/pj3.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:bool_bits_gemm -s 60 -c 1 -o gpurun_out/prof_bits16k $P warshall_bits16k --reps 1 > gpurun_out/ncu_pj3.log 2>&1
ls -la gpurun_out/*.ncu-rep | tail -4
