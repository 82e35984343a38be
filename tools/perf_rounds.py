"""Per-round phase-3 time of the C5 closure (n = 32768), from the live trace
(smx_fw_trace_*): shows which rounds run below the steady-state rate.

    python tools/perf_rounds.py [n]
"""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import _native, engines, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
lib = _native.lib()
(t,) = workloads.make_inputs(workloads.CONFIGS["c5_fw_u16"], n)
src = torch.from_numpy(t).cuda()
w = torch.empty_like(src)
for rep in range(2):
    w.copy_(src)
    torch.cuda.synchronize()
    cap = 1024
    lib.smx_fw_trace_arm(cap)
    engines.lane_close_(w, n, 16, True)
    torch.cuda.synchronize()
    ms = (ctypes.c_float * cap)()
    cells = (ctypes.c_longlong * cap)()
    k = lib.smx_fw_trace_read(ms, cells, cap)
rates = [cells[i] / (ms[i] / 1e3) for i in range(k) if cells[i] > 0]
print(json.dumps({"n": n, "rounds": len(rates), "rate_first8": [round(r / 1e12, 2) for r in rates[:8]],
                  "rate_median": sorted(rates)[len(rates) // 2] / 1e12,
                  "rate_last4": [round(r / 1e12, 2) for r in rates[-4:]]}))
