"""Host-buffer closure: serial copy-in / closure / copy-out against the
streamed smx_fw_host_u16 (AntidistMatrix.closure_of_host), same input.

    python tools/perf_host_fw.py [n ...]
Prints one JSON line per n: device-only closure time, the serial host path,
the streamed host path (ms, wall clock with synchronize), and whether the
streamed result equals the device closure bit for bit.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import AntidistMatrix, workloads  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    best = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best.append(time.perf_counter() - t0)
    return min(best) * 1e3, sum(best) / len(best) * 1e3


def main():
    ns = [int(x) for x in sys.argv[1:]] or [8192, 32768]
    cfg = workloads.CONFIGS["c5_fw_u16"]
    for n in ns:
        (t,) = workloads.make_inputs(cfg, n)
        pinned = torch.from_numpy(t).pin_memory()
        out = torch.empty_like(pinned).pin_memory()
        dev_in = pinned.cuda()
        reps = 2 if n >= 16384 else 5

        def device_only():
            return AntidistMatrix(n, n, 16, dev_in).transitive_closure()

        def serial():
            m = AntidistMatrix(n, n, 16, pinned.to("cuda", non_blocking=True))
            out.copy_(m.transitive_closure()._data, non_blocking=True)

        def streamed():
            AntidistMatrix.closure_of_host(pinned, 16, out=out)

        d = timed(device_only, reps)
        s = timed(serial, reps)
        st = timed(streamed, reps + 1)
        ref = device_only().data
        streamed()
        torch.cuda.synchronize()
        same = bool((out.numpy() == ref).all())
        print(json.dumps({"n": n, "device_ms": d, "serial_host_ms": s, "streamed_host_ms": st,
                          "bit_exact_vs_device": same,
                          "pcie_gb": 2 * pinned.numel() * 2 / 1e9}), flush=True)


if __name__ == "__main__":
    main()
