"""C1 (Boolean 1024^3) on E2M1 nibble operands (tcgen05 kind::mxf4) against
byte operands (kind::i8), development aid: the split-K pair kernel alone
replayed from a graph (one product per launch and 16 per launch), and the
public product (unpack + kernel) with smx_set_tc_f4 on / off.  Prints one
JSON object."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import BoolMatrix, _native, batch  # noqa: E402

lib = _native.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
nb = 16


def graph_time(fn, it=20, reps=10):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(it):
                fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / (it * reps)


def t_of(fn, it=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / it


a8 = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda")
peak = 2 * 8192 ** 3 / t_of(lambda: torch._int_mm(a8, a8.t()), 10, 2)
del a8
res = {"n": n, "int8_peak": peak}
sp = _native.stream_ptr
for rows in (n, nb * n):
    A8 = (torch.rand((rows, n), device="cuda") < 0.05).to(torch.uint8)
    Bt8 = (torch.rand((rows, n), device="cuda") < 0.05).to(torch.uint8)
    A4 = torch.randint(0, 256, (rows, n // 2), dtype=torch.uint8, device="cuda") & 0x22
    Bt4 = torch.randint(0, 256, (rows, n // 2), dtype=torch.uint8, device="cuda") & 0x22
    C = torch.zeros((rows, n // 32), dtype=torch.int32, device="cuda")
    if rows == n:
        f8 = lambda: lib.smx_bool_gemm_i8(A8.data_ptr(), Bt8.data_ptr(), None, C.data_ptr(), n, n, n, n, n,  # noqa
                                          n // 32, 0, sp())
        f4 = lambda: lib.smx_bool_gemm_f4(A4.data_ptr(), Bt4.data_ptr(), C.data_ptr(), n, n, n, n // 2, n // 2,  # noqa
                                          n // 32, 0, sp())
        tag, per = "single", 1
    else:
        f8 = lambda: lib.smx_bool_gemm_i8_batched(A8.data_ptr(), Bt8.data_ptr(), C.data_ptr(), nb, n, n, n, n, n,  # noqa
                                                  n // 32, 0, sp())
        f4 = lambda: lib.smx_bool_gemm_f4_batched(A4.data_ptr(), Bt4.data_ptr(), C.data_ptr(), nb, n, n, n,  # noqa
                                                  n // 2, n // 2, n // 32, 0, sp())
        tag, per = f"batch{nb}", nb
    for name, f in (("i8", f8), ("f4", f4)):
        t = graph_time(f, 20 if per == 1 else 5) / per
        res[f"{tag}_{name}_us"] = t * 1e6
        res[f"{tag}_{name}_frac_int8_peak"] = 2 * n ** 3 / t / peak
    del A8, Bt8, A4, Bt4, C
# batched nibble products: K slices x ring depth
A4 = torch.randint(0, 256, (nb * n, n // 2), dtype=torch.uint8, device="cuda") & 0x22
Bt4 = torch.randint(0, 256, (nb * n, n // 2), dtype=torch.uint8, device="cuda") & 0x22
C = torch.zeros((nb * n, n // 32), dtype=torch.int32, device="cuda")
for ks in (1, 2, 4):
    for stages in ((2, 3) if ks != 4 else (2,)):
        o_ks, o_st = lib.smx_set_tc_batch_ks(ks), lib.smx_set_tc_f4_batch_stages(stages)
        f = lambda: lib.smx_bool_gemm_f4_batched(A4.data_ptr(), Bt4.data_ptr(), C.data_ptr(), nb, n, n, n,  # noqa
                                                 n // 2, n // 2, n // 32, 0, sp())
        res[f"batch{nb}_f4_ks{ks}_st{stages}_us"] = graph_time(f, 5) / nb * 1e6
        lib.smx_set_tc_batch_ks(o_ks)
        lib.smx_set_tc_f4_batch_stages(o_st)
A8 = (torch.rand((nb * n, n), device="cuda") < 0.05).to(torch.uint8)
for ks in (1, 2, 4):
    o_ks = lib.smx_set_tc_batch_ks(ks)
    f = lambda: lib.smx_bool_gemm_i8_batched(A8.data_ptr(), A8.data_ptr(), C.data_ptr(), nb, n, n, n, n, n,  # noqa
                                             n // 32, 0, sp())
    res[f"batch{nb}_i8_ks{ks}_us"] = graph_time(f, 5) / nb * 1e6
    lib.smx_set_tc_batch_ks(o_ks)
o_pair = lib.smx_set_tc_pair(3)
f = lambda: lib.smx_bool_gemm_f4(A4.data_ptr(), Bt4.data_ptr(), C.data_ptr(), n, n, n, n // 2, n // 2,  # noqa
                                 n // 32, 0, sp())
res["single_f4_ks4_us"] = graph_time(f, 20) * 1e6
lib.smx_set_tc_pair(o_pair)
del A4, Bt4, C, A8
# the plain kernel (automatic tile width) at throughput shapes
for nn in (2048, 4096, 8192):
    A8 = (torch.rand((nn, nn), device="cuda") < 0.05).to(torch.uint8)
    A4 = torch.randint(0, 256, (nn, nn // 2), dtype=torch.uint8, device="cuda") & 0x22
    C = torch.zeros((nn, nn // 32), dtype=torch.int32, device="cuda")
    f8 = lambda: lib.smx_bool_gemm_i8(A8.data_ptr(), A8.data_ptr(), None, C.data_ptr(), nn, nn, nn, nn, nn,  # noqa
                                      nn // 32, 0, sp())
    f4 = lambda: lib.smx_bool_gemm_f4(A4.data_ptr(), A4.data_ptr(), C.data_ptr(), nn, nn, nn, nn // 2, nn // 2,  # noqa
                                      nn // 32, 0, sp())
    for name, f in (("i8", f8), ("f4", f4)):
        t = graph_time(f, 10 if nn < 8192 else 3, 5)
        res[f"n{nn}_{name}_us"] = t * 1e6
        res[f"n{nn}_{name}_frac_int8_peak"] = 2 * nn ** 3 / t / peak
    del A8, A4, C
rng = np.random.default_rng(1)
ma = BoolMatrix.from_numpy(rng.random((n, n)) < 0.05)
mb = BoolMatrix.from_numpy(rng.random((n, n)) < 0.05)
As = [BoolMatrix.from_numpy(rng.random((n, n)) < 0.05) for _ in range(nb)]
Bs = [BoolMatrix.from_numpy(rng.random((n, n)) < 0.05) for _ in range(nb)]
old = lib.smx_set_tc_f4(1)
for f in (1, 0):
    lib.smx_set_tc_f4(f)
    res[f"public_f4={f}_us"] = t_of(lambda: ma * mb) * 1e6
    res[f"bool_mul_many_f4={f}_us_per_product"] = t_of(lambda: batch.bool_mul_many(As, Bs), 10, 3) / nb * 1e6
lib.smx_set_tc_f4(old)
print(json.dumps(res))
