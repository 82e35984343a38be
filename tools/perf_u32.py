"""u32 lanes on the packed kernel (development aid): C4-size closure and a
4096^3 product, packed vs register-staged, per pivot block.  One JSON line."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_08743_b200 import DistMatrix, _native, workloads  # noqa: E402

lib = _native.lib()
S32 = (1 << 32) - 1


def timeit(fn, iters, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3


n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
(t16,) = workloads.make_inputs(workloads.CONFIGS["c4_fw_u16"], n)
d32 = np.where(t16 == 0, S32, 65535 - t16.astype(np.uint64)).astype(np.uint32)
src = DistMatrix(n, n, 32, d32)
res = {"n": n}
ref = None
for packed in (1, 0):
    for blk in (0, 128, 256):
        old_p = lib.smx_set_fw_packed(packed)
        old_b = lib.smx_set_fw_block(blk)
        try:
            m = src.copy()

            def run():
                m._data.copy_(src._data)
                m.transitive_close()
            t = timeit(run, 3)
            out = m.data
            if ref is None:
                ref = out
            res[f"fw_packed{packed}_blk{blk}"] = {"s": t, "cells_per_s": n ** 3 / t, "same": bool(np.array_equal(out, ref))}
        finally:
            lib.smx_set_fw_packed(old_p)
            lib.smx_set_fw_block(old_b)
rng = np.random.default_rng(1)
m = 4096
for name, wmax in (("bounded", 1000), ("general", 1 << 31)):
    a = np.where(rng.random((m, m)) < 0.1, rng.integers(1, wmax, (m, m), dtype=np.uint64), S32).astype(np.uint32)
    A = DistMatrix(m, m, 32, a)
    for packed in (1, 0):
        old_p = lib.smx_set_fw_packed(packed)
        try:
            t = timeit(lambda: A * A, 5)
        finally:
            lib.smx_set_fw_packed(old_p)
        res[f"mul4096_{name}_packed{packed}"] = {"s": t, "cells_per_s": m ** 3 / t}
print(json.dumps(res))
