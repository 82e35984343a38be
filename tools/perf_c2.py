"""Bit Warshall closure (C2 generator, mean out-degree 2) at 2048-16384:
the persistent one-launch closure against the blocked schedule."""
import json
import sys

import torch

sys.path.insert(0, '.')
from paper_1705_08743_b200 import BoolMatrix, _native, engines, workloads  # noqa: E402

lib = _native.lib()
cfg = workloads.CONFIGS["c2_bool_warshall"]
for n in [int(x) for x in sys.argv[1:]] or (2048, 4096, 8192, 16384):
    (t,) = workloads.make_inputs(cfg, n)
    m = BoolMatrix.from_numpy(t)
    rec = {"n": n}
    for mode in ("b128", "b256", "b512", 1):
        old = lib.smx_set_bool_persistent(1 if mode == 1 else 0)
        oldb = lib.smx_set_bool_block(int(mode[1:]) if mode != 1 else 0)
        for _ in range(3):
            engines.bool_closure_bits(m)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 20 if n <= 4096 else 5
        s.record()
        for _ in range(it):
            engines.bool_closure_bits(m)
        e.record()
        torch.cuda.synchronize()
        rec["persistent_ms" if mode == 1 else f"blocked_{mode}_ms"] = s.elapsed_time(e) / it
        lib.smx_set_bool_persistent(old)
        lib.smx_set_bool_block(oldb)
    print(json.dumps(rec), flush=True)
