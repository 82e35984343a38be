"""from_edges at C5 size (n = 32768, density 0.02: ~21.5M weighted edges)
through the public call, split into host validation, the edge upload and
the device fill + scatter (development aid).  Prints one JSON object."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import AntidistMatrix, _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
rng = np.random.default_rng(5)
m = int(0.02 * n * n)
edges = np.stack([rng.integers(0, n, m), rng.integers(0, n, m), rng.integers(1, 1001, m)], axis=1).astype(np.int64)
res = {"n": n, "edges": m}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mat = AntidistMatrix.from_edges(n, edges, 16)
    torch.cuda.synchronize()
    res[f"public_s_{rep}"] = time.perf_counter() - t0
    del mat
dev_edges = torch.from_numpy(edges).cuda()
data = torch.empty((n, n), dtype=torch.uint16, device="cuda")
lib = _native.lib()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    s.record()
    _native.check(lib.smx_from_edges(dev_edges.data_ptr(), m, data.data_ptr(), n, n, 2, _native.SMX_ANTI,
                                     _native.stream_ptr()), "from_edges")
    e.record()
    torch.cuda.synchronize()
res["device_ms"] = s.elapsed_time(e)
res["device_edges_per_s"] = m / (s.elapsed_time(e) / 1e3)
print(json.dumps(res))
