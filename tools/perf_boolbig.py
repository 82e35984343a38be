"""Boolean closure at 4096/8192/16384: bit-packed vs tensor-core path (development aid)."""
import sys, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1705_08743_b200 import BoolMatrix, engines
def timeit(fn, iters=3, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters
res = {}
rng = np.random.default_rng(0)
for n in (4096, 8192, 16384):
    m = BoolMatrix.from_numpy(rng.random((n, n), dtype=np.float32) < 2.0 / n)
    for eng in ("bool_closure_bits", "bool_closure_tc"):
        res[f"{eng}_{n}_ms"] = timeit(lambda: getattr(engines, eng)(m))
print(json.dumps(res, indent=1))
