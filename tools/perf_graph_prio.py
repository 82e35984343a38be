"""Eager vs graph replay of the FW closure, per side-stream variant (development aid)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1705_08743_b200 import _native, engines, workloads

lib = _native.lib()
def timeit(fn, iters, warm=1):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3
res = {}
for n in [int(x) for x in (sys.argv[1:] or ["8192"])]:
    cfg = workloads.CONFIGS["c4_fw_u16" if n <= 8192 else "c5_fw_u16"]
    (T,) = workloads.make_inputs(cfg, n)
    src = torch.from_numpy(T).cuda(); w = src.clone()
    def f():
        w.copy_(src); engines.lane_close_(w, n, 16, True)
    for graphs in (0, 1):
        for lite in (0, 1):
            lib.smx_set_graphs(graphs); lib.smx_set_fw_side_lite(lite)
            res[f"n{n}_graphs{graphs}_lite{lite}"] = f"{n**3 / timeit(f, 3 if n <= 8192 else 1, 1):.4e}"
    lib.smx_set_graphs(1); lib.smx_set_fw_side_lite(0)
print(json.dumps(res, indent=1))
