"""C1 (Boolean 1024^3) tensor-core kernel against its floors.

Back-to-back launches timed with CUDA events on the launching stream:
  null      torch.cuda._sleep(0): the launch floor of any kernel here
  int_mm    torch._int_mm (cuBLAS int8) at 1024^3: the library baseline
  tc        smx_bool_gemm_i8 (our tcgen05 kernel, bytes in, bits out), per
            output tile width (bn0 = automatic), and the split-K CTA pair
  tc_graph  the same, 20 launches per CUDA graph replay
  public    BoolMatrix.__mul__ (unpack + PDL kernel, graph replay)
Prints one JSON object.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1705_08743_b200 import BoolMatrix, _native, workloads  # noqa: E402


def timeit(fn, iters=400, warm=50):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def graphed(fn, per=20):
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(per):
                fn()
    return lambda: g.replay(), per


def main():
    lib = _native.lib()
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    dev = torch.device("cuda")
    res = {"n": n}
    res["null_us"] = timeit(lambda: torch.cuda._sleep(0))
    f, per = graphed(lambda: torch.cuda._sleep(0))
    res["null_graph_us"] = timeit(f, 50, 5) / per
    a8 = torch.randint(-127, 127, (n, n), dtype=torch.int8, device=dev)
    b8 = torch.randint(-127, 127, (n, n), dtype=torch.int8, device=dev)
    res["int_mm_us"] = timeit(lambda: torch._int_mm(a8, b8.t()))
    f, per = graphed(lambda: torch._int_mm(a8, b8.t()))
    res["int_mm_graph_us"] = timeit(f, 50, 5) / per
    A = (torch.rand((n, n), device=dev) < 0.05).to(torch.uint8)
    Bt = (torch.rand((n, n), device=dev) < 0.05).to(torch.uint8)
    out = torch.zeros((n, n // 32), dtype=torch.int32, device=dev)

    def tc():
        _native.check(lib.smx_bool_gemm_i8(A.data_ptr(), Bt.data_ptr(), None, out.data_ptr(), n, n, n, n, n,
                                           n // 32, 0, _native.stream_ptr(dev)), "tc")
    old = lib.smx_set_tc_tile_n(0)
    old_pair = lib.smx_set_tc_pair(0)
    for pair, bn in ((0, 0), (0, 64), (0, 128), (0, 256), (2, 0), (3, 0)):
        lib.smx_set_tc_pair(pair)
        lib.smx_set_tc_tile_n(bn)
        key = {0: f"tc_bn{bn}", 2: "tc_pair", 3: "tc_quad"}[pair]
        res[f"{key}_us"] = timeit(tc)
        f, per = graphed(tc)
        res[f"{key}_graph_us"] = timeit(f, 50, 5) / per
    lib.smx_set_tc_tile_n(old)
    lib.smx_set_tc_pair(old_pair)
    res["tc_us"], res["tc_graph_us"] = res["tc_bn0_us"], res["tc_bn0_graph_us"]
    if n == 1024:
        a, b = workloads.make_inputs(workloads.CONFIGS["c1_bool_mul"])
        ma, mb = BoolMatrix.from_numpy(a), BoolMatrix.from_numpy(b)
        res["public_us"] = timeit(lambda: ma * mb)
    res["ops"] = 2 * n ** 3
    res["tc_frac_of_int_mm_rate"] = res["int_mm_us"] / res["tc_us"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
