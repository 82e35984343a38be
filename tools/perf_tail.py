"""Wave quantisation of the packed phase-3 kernel: K = 256 products of
128*mt x 256 by 256 x 8192 (64 column tiles, so 64 * mt CTAs on 444 slots),
device time per product from graph replay, against mt.  Development aid."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import _native, engines  # noqa: E402

lib = _native.lib()
rng = np.random.default_rng(5)
N, K = 8192, 256
out = []
for mt in (55, 60, 62, 65, 69, 70, 76, 104, 111, 112):
    M = 128 * mt
    a = torch.from_numpy((65535 - rng.integers(1, 1000, (M, K))).astype(np.uint16)).cuda()
    b = torch.from_numpy((65535 - rng.integers(1, 1000, (K, N))).astype(np.uint16)).cuda()
    c = torch.empty((M, N), dtype=torch.uint16, device="cuda")
    f = lambda: engines.lane_mul(a, b, K, 16, True, c)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 20 / 1e3
    out.append({"mt": mt, "ctas": 64 * mt, "waves_444": 64 * mt / 444, "us": t * 1e6,
                "tcells_per_s": M * N * K / t / 1e12, "us_per_wave_equiv": t * 1e6 / (64 * mt / 444)})
    print(json.dumps(out[-1]), flush=True)
