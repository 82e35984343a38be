set -x
NCU=/usr/local/cuda/bin/ncu
python bench.py > gpurun_out/bench_r01_i.jsonl 2> gpurun_out/bench_r01_i.err
B32="python bench.py --steps 1 --warmup 1 --no-secondary --no-cpu"
$B32 > gpurun_out/plain_b32.log 2>&1 && $NCU --set full --clock-control none --import-source on -k regex:packed_gemm -s 41 -c 1 -o gpurun_out/prof_fw32k_packed_3b_i $B32 > gpurun_out/ncu_b32full.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_fw32768_r1i.csv $B32 > gpurun_out/ncu_b32list.log 2>&1
ls -la gpurun_out | tail -3
