set -x
NCU=/usr/local/cuda/bin/ncu
P="python tools/profile_kernels.py"
$P fw8k --reps 1 > gpurun_out/p4.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:packed_gemm -s 10 -c 1 -o gpurun_out/prof_fw8k_packed $P fw8k --reps 1 > gpurun_out/ncu_p4.log 2>&1
ls -la gpurun_out/ | tail -5
