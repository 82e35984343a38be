"""Side-chain (3a + pivot + row panel) span vs phase-3 span per round, from a
build with -DSMX_TRACE_SIDE (development aid)."""
import ctypes, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1705_08743_b200 import _native, engines, workloads
lib = _native.lib()
for n in [int(x) for x in (sys.argv[1:] or ["8192"])]:
    (T,) = workloads.make_inputs(workloads.CONFIGS["c4_fw_u16" if n <= 8192 else "c5_fw_u16"], n)
    src = torch.from_numpy(T).cuda(); w = src.clone()
    for rep in range(2):
        w.copy_(src); torch.cuda.synchronize()
        cap = 1024
        lib.smx_fw_trace_arm(cap)
        engines.lane_close_(w, n, 16, True); torch.cuda.synchronize()
        ms = (ctypes.c_float * cap)(); cells = (ctypes.c_longlong * cap)()
        k = lib.smx_fw_trace_read(ms, cells, cap)
    side = [ms[i] for i in range(k) if cells[i] == -1]
    p3 = [ms[i] for i in range(k) if cells[i] >= 0]
    parts = {name: [ms[i] for i in range(k) if cells[i] == code] for code, name in ((-2, "3a"), (-3, "pivot"), (-4, "row_panel"))}
    pp = {f"pivot_step{i}": [ms[j] for j in range(k) if cells[j] == -10 - i] for i in range(8)}
    if any(pp.values()):      # -DSMX_TRACE_PIVOT_PARTS: the 2 x 2 recursion's steps
        print(json.dumps({"n": n, **{f"{name}_ms_mean": sum(v) / max(len(v), 1) for name, v in pp.items()}}))
    if any(parts.values()):   # -DSMX_TRACE_SIDE_PARTS
        print(json.dumps({"n": n, **{f"{name}_ms_mean": sum(v) / max(len(v), 1) for name, v in parts.items()}}))
    print(json.dumps({"n": n, "rounds": len(p3), "side_ms_mean": sum(side) / max(len(side), 1),
                      "side_ms_max": max(side) if side else None, "p3_ms_mean": sum(p3) / max(len(p3), 1),
                      "side_longer_than_p3": sum(1 for a, b in zip(side, p3) if a > b)}))
