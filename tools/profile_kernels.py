"""Small, deterministic launches of each hot kernel for ncu captures."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1705_08743_b200 import BoolMatrix, engines, workloads

ap = argparse.ArgumentParser()
ap.add_argument("which", choices=["gemm_u16", "gemm_u8", "tc", "bits", "fw8k", "warshall_bits", "warshall_tc",
                                  "tc8k", "warshall_bits16k"])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
if a.which in ("gemm_u16", "gemm_u8"):
    cfg = workloads.CONFIGS["c3_mul_u16" if a.which == "gemm_u16" else "c3_mul_u8"]
    A, B = workloads.make_inputs(cfg)
    ta, tb = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty_like(ta)
    for _ in range(a.reps):
        engines.lane_mul(ta, tb, cfg.n, cfg.width, True, out)
elif a.which in ("tc", "bits"):
    A, B = workloads.make_inputs(workloads.CONFIGS["c1_bool_mul"])
    ma, mb = BoolMatrix.from_numpy(A), BoolMatrix.from_numpy(B)
    fn = engines.bool_mul_tc if a.which == "tc" else engines.bool_mul_bits
    for _ in range(a.reps):
        fn(ma, mb)
elif a.which == "fw8k":
    (T,) = workloads.make_inputs(workloads.CONFIGS["c4_fw_u16"])
    t = torch.from_numpy(T).cuda()
    for _ in range(a.reps):
        engines.lane_close_(t.clone(), 8192, 16, True)
elif a.which == "tc8k":
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    n = 8192
    A = (torch.rand((n, n), device="cuda") < 0.05).to(torch.uint8)
    Bt = (torch.rand((n, n), device="cuda") < 0.05).to(torch.uint8)
    out = torch.zeros((n, n // 32), dtype=torch.int32, device="cuda")
    for _ in range(a.reps):
        _native.check(lib.smx_bool_gemm_i8(A.data_ptr(), Bt.data_ptr(), None, out.data_ptr(), n, n, n, n, n,
                                           n // 32, 0, _native.stream_ptr()), "tc")
elif a.which == "warshall_bits16k":
    import numpy as np
    n = 16384
    m = BoolMatrix.from_numpy(np.random.default_rng(0).random((n, n), dtype=np.float32) < 2.0 / n)
    for _ in range(a.reps):
        engines.bool_closure_bits(m)
else:
    (T,) = workloads.make_inputs(workloads.CONFIGS["c2_bool_warshall"])
    m = BoolMatrix.from_numpy(T)
    fn = engines.bool_closure_bits if a.which == "warshall_bits" else engines.bool_closure_tc
    for _ in range(a.reps):
        fn(m)
torch.cuda.synchronize()
print("ok")
