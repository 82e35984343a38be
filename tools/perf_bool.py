"""Boolean engine timings: TC i8 GEMM at several n vs torch._int_mm int8 peak (development aid)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1705_08743_b200 import BoolMatrix, _native, engines, workloads

lib = _native.lib()

def timeit(fn, iters, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3

res = {}
a8 = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda")
b8 = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda")
t = timeit(lambda: torch._int_mm(a8, b8.t()), 10)
res["torch_int_mm_8192_ops_per_s"] = 2 * 8192**3 / t
for n in (1024, 2048, 4096, 8192, 16384):
    A = (torch.rand((n, n), device="cuda") < 0.05).to(torch.uint8)
    Bt = (torch.rand((n, n), device="cuda") < 0.05).to(torch.uint8)
    out = torch.zeros((n, n // 32), dtype=torch.int32, device="cuda")
    f = lambda: _native.check(lib.smx_bool_gemm_i8(A.data_ptr(), Bt.data_ptr(), None, out.data_ptr(), n, n, n, n, n, n // 32, 0, _native.stream_ptr()), "tc")
    t = timeit(f, 20 if n <= 4096 else 5)
    res[f"tc_gemm_{n}"] = {"us": t * 1e6, "ops_per_s": 2 * n**3 / t}
    outb = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    f = lambda: _native.check(lib.smx_bool_gemm_i8(A.data_ptr(), Bt.data_ptr(), outb.data_ptr(), None, n, n, n, n, n, n, 0, _native.stream_ptr()), "tc")
    t = timeit(f, 20 if n <= 4096 else 5)
    res[f"tc_gemm_bytesout_{n}"] = {"us": t * 1e6, "ops_per_s": 2 * n**3 / t}
cfg = workloads.CONFIGS["c1_bool_mul"]; A, B = workloads.make_inputs(cfg)
ma, mb = BoolMatrix.from_numpy(A), BoolMatrix.from_numpy(B)
for eng in ("bool_mul_tc", "bool_mul_bits"):
    fn = getattr(engines, eng)
    res[f"c1_{eng}_us"] = timeit(lambda: fn(ma, mb), 50, 5) * 1e6
cfg = workloads.CONFIGS["c2_bool_warshall"]; (T,) = workloads.make_inputs(cfg)
m = BoolMatrix.from_numpy(T)
for eng in ("bool_closure_tc", "bool_closure_bits"):
    fn = getattr(engines, eng)
    res[f"c2_{eng}_us"] = timeit(lambda: fn(m), 10, 2) * 1e6
print(json.dumps(res, indent=1))

# CUDA-graph replay of the C2 closure: separates GPU time from host launch cost
ws = torch.empty(max(1, lib.smx_bool_warshall_workspace_bytes(m.rows, m.stride_words)), dtype=torch.uint8, device="cuda")
work = m._words.clone()
st = torch.cuda.Stream()
def c2_call():
    _native.check(lib.smx_bool_warshall_bits(work.data_ptr(), m.rows, m.stride_words, ws.data_ptr(), ws.numel(),
                                            torch.cuda.current_stream().cuda_stream), "warshall")
with torch.cuda.stream(st):
    c2_call(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        c2_call()
torch.cuda.synchronize()
res2 = {"c2_bits_eager_us": timeit(c2_call, 20, 3) * 1e6, "c2_bits_graph_us": timeit(g.replay, 20, 3) * 1e6}
print(json.dumps(res2, indent=1))
