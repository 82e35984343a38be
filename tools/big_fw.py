"""Single-GPU closures beyond C5's n = 32768 (the HBM-capacity end of the
path): the C5 generator at n = 49152 / 65536 (4.5 / 8 GiB of u16), one timed
closure, and two size-independent checks -- closing the closure again
changes nothing (idempotence), and the host-buffer closure (smx_fw_host_u16)
gives the same bytes.

    python tools/big_fw.py [n ...]
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import AntidistMatrix, workloads  # noqa: E402


def main():
    cfg = workloads.CONFIGS["c5_fw_u16"]
    for n in [int(x) for x in sys.argv[1:]] or [65536]:
        t0 = time.perf_counter()
        (host,) = workloads.make_inputs(cfg, n)
        gen_s = time.perf_counter() - t0
        dev_in = torch.from_numpy(host).cuda()
        m = AntidistMatrix(n, n, 16, dev_in)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        c = m.transitive_closure()
        e.record()
        torch.cuda.synchronize()
        secs = s.elapsed_time(e) / 1e3
        again = c.transitive_closure()
        idem = bool(torch.equal(again._data, c._data))
        del again
        pinned = torch.from_numpy(host).pin_memory()
        out = torch.empty_like(pinned).pin_memory()
        t1 = time.perf_counter()
        AntidistMatrix.closure_of_host(pinned, 16, out=out)
        torch.cuda.synchronize()
        host_secs = time.perf_counter() - t1
        same = bool(torch.equal(out, c._data.cpu()))
        digest = hashlib.sha256(c._data.cpu().numpy().tobytes()).hexdigest()
        print(json.dumps({"n": n, "bytes": n * host.shape[1] * 2, "closure_s": secs,
                          "cells_per_s": n ** 3 / secs, "host_buffer_closure_s": host_secs,
                          "host_buffer_cells_per_s": n ** 3 / host_secs, "idempotent": idem,
                          "host_buffer_equals_device": same, "sha256": digest,
                          "generate_s": gen_s}), flush=True)
        del m, c, dev_in, pinned, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
