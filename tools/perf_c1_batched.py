"""C1-shaped Boolean products (1024^3) one per call against many per launch
(development aid): the public product in a loop, bool_mul_many (the batched
split-K pair on the tensor cores), and the batched kernel alone on unpacked
operands replayed from a graph; per-product device time and the fraction of
the measured int8 peak.  Prints one JSON object."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import BoolMatrix, _native, batch, workloads  # noqa: E402

lib = _native.lib()
n, nb = 1024, int(sys.argv[1]) if len(sys.argv) > 1 else 16


def t_of(fn, it=20, warm=3):
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
rng = np.random.default_rng(1)
As = [BoolMatrix.from_numpy(rng.random((n, n)) < 0.05) for _ in range(nb)]
Bs = [BoolMatrix.from_numpy(rng.random((n, n)) < 0.05) for _ in range(nb)]
res = {"n": n, "batch": nb, "int8_peak": peak}
t = t_of(lambda: [a * b for a, b in zip(As, Bs)], 5, 2)
res["public_loop_us_per_product"] = t / nb * 1e6
t = t_of(lambda: batch.bool_mul_many(As, Bs), 10, 3)
res["bool_mul_many_us_per_product"] = t / nb * 1e6
A8 = (torch.rand((nb * n, n), device="cuda") < 0.05).to(torch.uint8)
Bt8 = (torch.rand((nb * n, n), device="cuda") < 0.05).to(torch.uint8)
C = torch.zeros((nb * n, n // 32), dtype=torch.int32, device="cuda")


def kern():
    _native.check(lib.smx_bool_gemm_i8_batched(A8.data_ptr(), Bt8.data_ptr(), C.data_ptr(), nb, n, n, n, n, n,
                                               n // 32, 0, _native.stream_ptr()), "batched")


g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    kern()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        for _ in range(10):
            kern()
t = t_of(lambda: g.replay(), 10, 2) / 10
res["batched_kernel_us_per_product"] = t / nb * 1e6
res["batched_kernel_frac_of_int8_peak"] = 2 * n ** 3 * nb / t / peak
old = lib.smx_set_tc_batch_ks(4)
g4 = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    kern()
    torch.cuda.synchronize()
    with torch.cuda.graph(g4, stream=st):
        for _ in range(10):
            kern()
lib.smx_set_tc_batch_ks(old)
t = t_of(lambda: g4.replay(), 10, 2) / 10
res["batched_ks4_us_per_product"] = t / nb * 1e6
res["batched_ks4_frac_of_int8_peak"] = 2 * n ** 3 * nb / t / peak
print(json.dumps(res))
