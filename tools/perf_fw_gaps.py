"""Where the main stream waits between phase-3 launches of a closure
(development aid): CUDA events around every phase-3 launch (smx_fw_trace_*),
the gap from one launch's end to the next one's begin, per round.  The
trace keeps the closure eager (no replay graph).  Prints one JSON object."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import _native, engines, workloads  # noqa: E402

lib = _native.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cfg = workloads.CONFIGS["c4_fw_u16" if n <= 8192 else "c5_fw_u16"]
(x,) = workloads.make_inputs(cfg, n)
src = torch.from_numpy(x).cuda()
w = torch.empty_like(src)
cap = 1024
for rep in range(3):
    w.copy_(src)
    torch.cuda.synchronize()
    lib.smx_fw_trace_arm(cap)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    engines.lane_close_(w, n, 16, True)
    e.record()
    torch.cuda.synchronize()
    b = (ctypes.c_float * cap)()
    en = (ctypes.c_float * cap)()
    k = lib.smx_fw_trace_offsets(b, en, cap)
    ms = (ctypes.c_float * cap)()
    cells = (ctypes.c_longlong * cap)()
    lib.smx_fw_trace_read(ms, cells, cap)
total = s.elapsed_time(e)
gaps = [b[i + 1] - en[i] for i in range(k - 1)]
res = {"n": n, "launches": k, "total_ms": total, "before_first_and_after_last_ms": total - en[k - 1],
       "phase3_ms": sum(en[i] - b[i] for i in range(k)), "gaps_ms_sum": sum(gaps),
       "gap_ms_mean": sum(gaps) / max(len(gaps), 1), "gap_ms_max": max(gaps) if gaps else None,
       "gaps_ms": [round(g, 4) for g in gaps]}
print(json.dumps(res))
