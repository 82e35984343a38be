"""Quick device timings of each engine (development aid; bench.py is the contract)."""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes
import numpy as np
import torch
from paper_1705_08743_b200 import _native, engines, workloads, BoolMatrix

def timeit(fn, iters=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3

def probe(one):
    lib = _native.lib()
    sink = torch.zeros(148*8*256, dtype=torch.int32, device="cuda")
    ipt = ctypes.c_longlong(0)
    blocks, threads, iters = 148*8, 256, 20000
    f = lambda: _native.check(lib.smx_int_issue_probe(sink.data_ptr(), blocks, threads, iters, one, ctypes.byref(ipt), _native.stream_ptr()), "probe")
    t = timeit(f, 3, 1)
    return blocks*threads*ipt.value/t

ap = argparse.ArgumentParser(); ap.add_argument("--gemm-only", action="store_true"); a = ap.parse_args()
res = {}
if not a.gemm_only:
    res["issue_2instr_per_s"] = probe(0); res["issue_1instr_per_s"] = probe(1)
for name in ("c3_mul_u16", "c3_mul_u8"):
    cfg = workloads.CONFIGS[name]; n = cfg.n
    A, B = workloads.make_inputs(cfg)
    ta, tb = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty_like(ta)
    t = timeit(lambda: engines.lane_mul(ta, tb, n, cfg.width, True, out))
    res[name] = dict(seconds=t, cells_per_s=n**3/t)
for nm, nfw in (("c4_fw_u16", 8192),):
    cfg = workloads.CONFIGS[nm]
    (T,) = workloads.make_inputs(cfg, nfw)
    tt = torch.from_numpy(T).cuda(); w = tt.clone()
    def f():
        w.copy_(tt); engines.lane_close_(w, nfw, 16, True)
    t = timeit(f, 3, 1)
    res[nm] = dict(n=nfw, seconds=t, cells_per_s=nfw**3/t)
if not a.gemm_only:
    cfg = workloads.CONFIGS["c1_bool_mul"]; A, B = workloads.make_inputs(cfg)
    ma, mb = BoolMatrix.from_numpy(A), BoolMatrix.from_numpy(B)
    t = timeit(lambda: ma * mb, 20, 3); res["c1_bool_mul_bits"] = dict(seconds=t, cells_per_s=1024**3/t)
    cfg = workloads.CONFIGS["c2_bool_warshall"]; (T,) = workloads.make_inputs(cfg)
    m = BoolMatrix.from_numpy(T)
    t = timeit(lambda: m.transitive_closure(), 5, 2); res["c2_warshall_bits"] = dict(seconds=t, cells_per_s=4096**3/t)
print(json.dumps(res, indent=1))
