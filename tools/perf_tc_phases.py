"""Phase breakdown of the C1 tensor-core kernel (development aid).

Arms smx_tc_trace_arm and runs the kernel (tile width argv[2], default 64)
at 1024^3 a few times; prints CTA 0's clock64 phases and the spread of every
CTA's globaltimer entry/exit.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1705_08743_b200 import _native  # noqa: E402

lib = _native.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
A = (torch.rand((n, n), device="cuda") < 0.05).to(torch.uint8)
Bt = (torch.rand((n, n), device="cuda") < 0.05).to(torch.uint8)
out = torch.zeros((n, n // 32), dtype=torch.int32, device="cuda")
buf = torch.zeros(16 + 2 * 4096, dtype=torch.int64, device="cuda")
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 64
pair = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # 2: the split-K CTA pair
old = lib.smx_set_tc_tile_n(variant)
old_pair = lib.smx_set_tc_pair(pair)


def run():
    _native.check(lib.smx_bool_gemm_i8(A.data_ptr(), Bt.data_ptr(), None, out.data_ptr(), n, n, n, n, n,
                                       n // 32, 0, _native.stream_ptr()), "tc")


for _ in range(20):
    run()
lib.smx_tc_trace_arm(buf.data_ptr())
res = []
for rep in range(5):
    buf.zero_()
    torch.cuda.synchronize()         # an idle GPU: no PDL predecessor to wait for
    run()
    torch.cuda.synchronize()
    b = buf.cpu().tolist()
    ph = b[:12]
    ctas = [(b[16 + 2 * i], b[17 + 2 * i]) for i in range(4096) if b[16 + 2 * i]]
    t0 = min(c[0] for c in ctas)
    res.append({
        "cycles_cta0": {"prologue": ph[1] - ph[0], "tma_issued": ph[2] - ph[0], "first_stage": ph[3] - ph[0],
                        "last_stage": ph[4] - ph[0], "mma_done": ph[5] - ph[0], "epilogue_done": ph[6] - ph[0],
                        "merged": (ph[7] - ph[0]) if ph[7] else None,
                        "pair_detail": {k: (ph[i] - ph[0]) if ph[i] else None for k, i in
                                        (("bits", 8), ("cluster_wait", 9), ("mbar_init", 10), ("tmem_alloc", 11))}},
        "ctas": len(ctas),
        "entry_spread_ns": max(c[0] for c in ctas) - t0,
        "first_exit_ns": min(c[1] for c in ctas) - t0,
        "last_exit_ns": max(c[1] for c in ctas) - t0,
    })
lib.smx_tc_trace_arm(None)
lib.smx_set_tc_tile_n(old)
lib.smx_set_tc_pair(old_pair)
print(json.dumps({"n": n, "tile_n": variant, "pair": pair, "runs": res[-2:]}, indent=1))
