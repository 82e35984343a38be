"""u16 closure time per pivot block size (smx_set_fw_block) at several n.

    python tools/perf_fw_blocks.py [n ...]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import _native, engines, workloads  # noqa: E402

lib = _native.lib()
cfg = workloads.CONFIGS["c4_fw_u16"]
for n in [int(x) for x in sys.argv[1:]] or [4096, 8192, 16384]:
    (x,) = workloads.make_inputs(cfg, n)
    src = torch.from_numpy(x).cuda()
    w = torch.empty_like(src)
    for blk in (0, 128, 256, 512):
        old = lib.smx_set_fw_block(blk)
        try:
            def close():
                w.copy_(src)
                engines.lane_close_(w, n, 16, True)
            for _ in range(2):
                close()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            it = 3 if n >= 16384 else 10
            s.record()
            for _ in range(it):
                close()
            e.record()
            torch.cuda.synchronize()
            sec = s.elapsed_time(e) / 1e3 / it
        finally:
            lib.smx_set_fw_block(old)
        print(json.dumps({"n": n, "block": blk or "auto", "ms": sec * 1e3, "cells_per_s": n ** 3 / sec}), flush=True)
