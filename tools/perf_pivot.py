"""Pivot kernels and the closures they bound: smx_fw_pivot at b = 128 / 256 /
512 on an idle GPU, and full u16 closures at n = 1024 .. 32768, with the
blocked pivot kernel (smx_set_fw_pivot_blocked(1)) and the register kernel (0).

    python tools/perf_pivot.py [n ...]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import _native, engines, workloads  # noqa: E402


def cuda_time(fn, iters, warm=2):
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


lib = _native.lib()
ns = [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096, 8192, 16384, 32768]
cfg = workloads.CONFIGS["c5_fw_u16"]
(t,) = workloads.make_inputs(cfg, 1024)
tile = torch.from_numpy(t).cuda()
for blocked in (0, 1):
    old = lib.smx_set_fw_pivot_blocked(blocked)
    try:
        for b in (128, 256, 512):
            work = tile.clone()
            f = lambda: _native.check(lib.smx_fw_pivot(work.data_ptr(), b, work.shape[1], 2, 0,  # noqa: E731
                                                       _native.stream_ptr()), "pivot")
            us = cuda_time(f, 20) * 1e6
            print(json.dumps({"blocked": blocked, "pivot_b": b, "us": us}), flush=True)
        for n in ns:
            (x,) = workloads.make_inputs(cfg, n)
            src = torch.from_numpy(x).cuda()
            w = torch.empty_like(src)

            def close():
                w.copy_(src)
                engines.lane_close_(w, n, 16, True)
            sec = cuda_time(close, 3 if n >= 16384 else 10)
            print(json.dumps({"blocked": blocked, "n": n, "ms": sec * 1e3, "cells_per_s": n ** 3 / sec}),
                  flush=True)
    finally:
        lib.smx_set_fw_pivot_blocked(old)
