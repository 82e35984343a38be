"""Public semiring products at C3 (4096^3) and neighbouring sizes: time per
product and cell-updates/s (development aid for the split-K choice).

    python tools/perf_products.py
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import engines, workloads  # noqa: E402


def cuda_time(fn, iters=10, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / iters


for name in ("c3_mul_u8", "c3_mul_u16"):
    cfg = workloads.CONFIGS[name]
    for n in (2048, 3072, 4096, 6144):
        a, b = workloads.make_inputs(cfg, n)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        res = torch.empty_like(ta)
        t = cuda_time(lambda: engines.lane_mul(ta, tb, n, cfg.width, True, res))
        print(json.dumps({"workload": name, "n": n, "ms": t * 1e3, "cells_per_s": n ** 3 / t}), flush=True)
