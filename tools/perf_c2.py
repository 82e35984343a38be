import json, sys, torch
sys.path.insert(0, '.')
from paper_1705_08743_b200 import BoolMatrix, engines, workloads
cfg = workloads.CONFIGS["c2_bool_warshall"]
for n in (2048, 4096, 8192, 16384):
    (t,) = workloads.make_inputs(cfg, n)
    m = BoolMatrix.from_numpy(t)
    for _ in range(3): engines.bool_closure_bits(m)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20 if n <= 4096 else 5
    s.record()
    for _ in range(it): engines.bool_closure_bits(m)
    e.record(); torch.cuda.synchronize()
    print(json.dumps({"n": n, "ms": s.elapsed_time(e) / it}), flush=True)
