"""Full-size determinism check: the C5 closure (n = 32768) under every schedule
switch and repeated runs must give one sha256 (development aid; writes JSON)."""
import hashlib, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1705_08743_b200 import _native, engines, workloads

lib = _native.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
cfg = workloads.CONFIGS["c5_fw_u16"]
(T,) = workloads.make_inputs(cfg, n)
src = torch.from_numpy(T).cuda()
res = {"n": n}
variants = [("default", {}), ("default_again", {}), ("lookahead_off", {"smx_set_fw_lookahead": 0}),
            ("register_phase3", {"smx_set_fw_packed": 0}), ("graphs_off", {"smx_set_graphs": 0}),
            ("block256", {"smx_set_fw_block": 256}), ("general_form", {"smx_set_bounded_fastpath": 0}),
            ("register_pivot", {"smx_set_fw_pivot_blocked": 0})]
for name, sw in variants:
    olds = {k: getattr(lib, k)(v) for k, v in sw.items()}
    try:
        w = src.clone()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        engines.lane_close_(w, n, 16, True)
        torch.cuda.synchronize()
        res[name] = {"sha256": hashlib.sha256(w.cpu().numpy().tobytes()).hexdigest()[:16],
                     "s": round(time.perf_counter() - t0, 3)}
    finally:
        for k, v in olds.items():
            getattr(lib, k)(v)
# the host-buffer closure (copies overlapped, ingest / egress products)
from paper_1705_08743_b200 import AntidistMatrix  # noqa: E402
pinned = torch.from_numpy(T).pin_memory()
torch.cuda.synchronize(); t0 = time.perf_counter()
_, out = AntidistMatrix.closure_of_host(pinned, 16)
torch.cuda.synchronize()
res["host_buffer"] = {"sha256": hashlib.sha256(out.numpy().tobytes()).hexdigest()[:16],
                      "s": round(time.perf_counter() - t0, 3)}
res["all_equal"] = len({v["sha256"] for k, v in res.items() if isinstance(v, dict)}) == 1
print(json.dumps(res, indent=1))
