"""Phase-3 share of an FW closure (trace events around each phase-3 launch) -- development aid."""
import ctypes, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_1705_08743_b200 import _native, engines, workloads

lib = _native.lib()
res = {}
for n in [int(x) for x in (sys.argv[1:] or ["8192"])]:
    cfg = workloads.CONFIGS["c4_fw_u16" if n <= 8192 else "c5_fw_u16"]
    (T,) = workloads.make_inputs(cfg, n)
    src = torch.from_numpy(T).cuda(); w = src.clone()
    for rep in range(3):
        w.copy_(src)
        torch.cuda.synchronize()
        rounds = 200
        lib.smx_fw_trace_arm(rounds)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); engines.lane_close_(w, n, 16, True); e.record(); torch.cuda.synchronize()
        ms = (ctypes.c_float * rounds)(); cells = (ctypes.c_longlong * rounds)()
        cnt = lib.smx_fw_trace_read(ms, cells, rounds)
        tot = s.elapsed_time(e)
        p3 = sum(ms[:cnt])
        res[f"n{n}_rep{rep}"] = {"total_ms": tot, "phase3_ms": p3, "share": p3 / tot, "launches": cnt,
                                 "phase3_cells_per_s": sum(cells[:cnt]) / (p3 / 1e3),
                                 "closure_cells_per_s": n**3 / (tot / 1e3)}
print(json.dumps(res, indent=1))

# pivot tile closure alone (public smx_fw_pivot), b = 128 and 256
for b in (128, 256):
    cfg = workloads.CONFIGS["c5_fw_u16"]
    (T,) = workloads.make_inputs(cfg, 4096)
    t = torch.from_numpy(T).cuda()
    ld = t.shape[1]
    def piv():
        _native.check(lib.smx_fw_pivot(t.data_ptr(), b, ld, 2, 0, _native.stream_ptr()), "pivot")
    for _ in range(3): piv()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): piv()
    e.record(); torch.cuda.synchronize()
    print(f"pivot b={b}: {s.elapsed_time(e) / 20 * 1e3:.1f} us")
