"""FW / GEMM timing matrix over the schedule switches (development aid)."""
import json, sys, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1705_08743_b200 import _native, engines, workloads

lib = _native.lib()

def timeit(fn, iters, warm=1):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3

res = {"variant": os.environ.get("SMX_GEMM_VARIANT", "0")}
for name in ("c3_mul_u16", "c3_mul_u8"):
    cfg = workloads.CONFIGS[name]; n = cfg.n
    A, B = workloads.make_inputs(cfg)
    ta, tb = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty_like(ta)
    t = timeit(lambda: engines.lane_mul(ta, tb, n, cfg.width, True, out), 10, 2)
    res[name] = n**3 / t
sizes = [int(x) for x in (sys.argv[1:] or ["8192"])]
for n in sizes:
    cfg = workloads.CONFIGS["c4_fw_u16" if n <= 8192 else "c5_fw_u16"]
    (T,) = workloads.make_inputs(cfg, n)
    src = torch.from_numpy(T).cuda(); w = src.clone()
    def f():
        w.copy_(src); engines.lane_close_(w, n, 16, True)
    variants = [(1, 1, 0, 0, 1), (1, 1, 0, 0, 0), (1, 0, 0, 0, 1)]
    if os.environ.get("PERF_FW_ALL"):
        variants += [(1, 1, 1, 0, 1), (1, 1, 0, 128, 1), (1, 1, 0, 256, 1), (1, 1, 0, 512, 1)]
    for fast, la, lite, blk, packed in variants:
        lib.smx_set_bounded_fastpath(fast); lib.smx_set_fw_lookahead(la); lib.smx_set_fw_side_lite(lite)
        lib.smx_set_fw_block(blk); lib.smx_set_fw_packed(packed)
        t = timeit(f, 3 if n <= 8192 else 1, 1)
        res[f"fw{n}_fast{fast}_la{la}_lite{lite}_b{blk}_packed{packed}"] = n**3 / t
    lib.smx_set_bounded_fastpath(1); lib.smx_set_fw_lookahead(1); lib.smx_set_fw_side_lite(0)
    lib.smx_set_fw_block(0); lib.smx_set_fw_packed(1)
print(json.dumps({k: (f"{v:.4e}" if isinstance(v, float) else v) for k, v in res.items()}))
