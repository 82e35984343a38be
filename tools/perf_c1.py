"""C1 (Boolean 1024^3) call-overhead breakdown (development aid)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1705_08743_b200 import BoolMatrix, _native, engines, workloads

lib = _native.lib()
A, B = workloads.make_inputs(workloads.CONFIGS["c1_bool_mul"])
ma, mb = BoolMatrix.from_numpy(A), BoolMatrix.from_numpy(B)

def timeit(fn, iters=200, warm=20):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3

res = {"public_us": timeit(lambda: ma * mb), "engine_us": timeit(lambda: engines.bool_mul_tc(ma, mb))}
out = torch.empty((1024, 32), dtype=torch.int32, device="cuda")
nb = lib.smx_bool_mul_tc_workspace_bytes(1024, 1024, 1024)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
st = _native.stream_ptr()
def direct():
    lib.smx_bool_mul_tc(ma._words.data_ptr(), mb._words.data_ptr(), out.data_ptr(), 1024, 1024, 1024,
                        ma.stride_words, mb.stride_words, 32, ws.data_ptr(), nb, st)
res["direct_c_call_us"] = timeit(direct)
g = torch.cuda.CUDAGraph()
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    direct(); torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s2):
        for _ in range(20): direct()
res["device_per_call_us (20 calls in one graph)"] = timeit(g.replay, 20, 3) / 20
print(json.dumps(res, indent=1))

# host-side cost per call (no sync inside the loop): if it exceeds the GPU
# time per call, the public call is host-bound
import time
for name, fn in (("public", lambda: ma * mb), ("engine", lambda: engines.bool_mul_tc(ma, mb)), ("direct", direct)):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(500): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"host_us_per_call {name}: {(t1 - t0) / 500 * 1e6:.2f}")
