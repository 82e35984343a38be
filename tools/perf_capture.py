"""First-call cost of graph capture vs eager launches for the closures (development aid)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1705_08743_b200 import _native, engines, workloads

lib = _native.lib()
res = {}
for n in [int(x) for x in (sys.argv[1:] or ["2048", "8192", "32768"])]:
    cfg = workloads.CONFIGS["c5_fw_u16"]
    (T,) = workloads.make_inputs(cfg, n)
    src = torch.from_numpy(T).cuda()
    for graphs in (1, 0):
        lib.smx_set_graphs(graphs)
        times = []
        for i in range(3):
            w = src.clone() if i == 0 else w   # first call: a fresh pointer
            w.copy_(src)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            engines.lane_close_(w, n, 16, True)
            torch.cuda.synchronize(); times.append((time.perf_counter() - t0) * 1e3)
        res[f"n{n}_graphs{graphs}_ms"] = [round(t, 2) for t in times]
    lib.smx_set_graphs(1)
print(json.dumps(res, indent=1))
