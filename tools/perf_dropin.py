"""The reference's literal call on a host array against the page-locked
host-buffer call and the device-resident closure (development aid):
    AntidistMatrix(n, n, 16, ndarray).transitive_closure().data
Prints one JSON object."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1705_08743_b200 import AntidistMatrix, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
cfg = workloads.CONFIGS["c5_fw_u16"]
(host,) = workloads.make_inputs(cfg, n)
res = {"n": n}


def timed(fn, reps=2, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


res["dropin_ms"] = timed(lambda: AntidistMatrix(n, n, 16, host).transitive_closure().data) * 1e3
work = host.copy()


def in_place():
    work[...] = host              # (host memcpy, outside the library call)
    AntidistMatrix(n, n, 16, work).transitive_close()


t_copy = timed(lambda: work.__setitem__(Ellipsis, host))
res["in_place_ms"] = (timed(in_place) - t_copy) * 1e3     # the refill subtracted
del work
pinned = torch.from_numpy(host).pin_memory()
out = torch.empty_like(pinned).pin_memory()
res["pinned_call_ms"] = timed(lambda: AntidistMatrix.closure_of_host(pinned, 16, out=out)) * 1e3
src = torch.from_numpy(host).cuda()
w = torch.empty_like(src)
m = AntidistMatrix(n, n, 16, w)


def dev():
    w.copy_(src)
    m.transitive_close()


res["device_ms"] = timed(dev) * 1e3
res["cells_per_s_dropin"] = n ** 3 / res["dropin_ms"] * 1e3
del pinned, out, src, w, m
torch.cuda.empty_cache()
# the product: (AntidistMatrix(n, n, 16, a) * AntidistMatrix(n, n, 16, b)).data
mcfg = workloads.CONFIGS["c5_mul_u16"] if "c5_mul_u16" in workloads.CONFIGS else None
if mcfg is not None:
    a, b = workloads.make_inputs(mcfg, n)
    res["mul_dropin_ms"] = timed(lambda: (AntidistMatrix(n, n, 16, a) * AntidistMatrix(n, n, 16, b)).data) * 1e3
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    res["mul_device_ms"] = timed(lambda: AntidistMatrix(n, n, 16, da) * AntidistMatrix(n, n, 16, db)) * 1e3
print(json.dumps(res))
