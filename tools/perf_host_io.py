"""Host-side I/O rates on the GPU box (development aid for the drop-in
host-buffer closure): memcpy pageable -> pinned with torch's CPU copy
(threads), cudaHostRegister / unregister of a user array, and H2D / D2H
bandwidth from pageable and pinned memory.  Prints one JSON object."""
import json
import os
import time

import numpy as np
import torch

GB = 2 ** 30
n = int(os.environ.get("SMX_IO_BYTES", str(2 * GB)))
res = {"bytes": n, "cpu_count": os.cpu_count(), "torch_threads": torch.get_num_threads()}
src = np.ones(n // 2, dtype=np.uint16)          # touched (resident) pageable array
t0 = time.perf_counter()
pin = torch.empty(n // 2, dtype=torch.int16, pin_memory=True)
res["pinned_alloc_s"] = time.perf_counter() - t0
for th in (1, 4, 8, torch.get_num_threads()):
    torch.set_num_threads(th)
    st = torch.from_numpy(src.view(np.int16))
    pin.copy_(st)
    t0 = time.perf_counter()
    for _ in range(3):
        pin.copy_(st)
    res[f"memcpy_to_pinned_gbs_t{th}"] = 3 * n / (time.perf_counter() - t0) / 1e9
dev = torch.empty(n // 2, dtype=torch.int16, device="cuda")
for name, h in (("pinned", pin), ("pageable", torch.from_numpy(src.view(np.int16)))):
    dev.copy_(h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        dev.copy_(h)
    torch.cuda.synchronize()
    res[f"h2d_{name}_gbs"] = 3 * n / (time.perf_counter() - t0) / 1e9
    t0 = time.perf_counter()
    for _ in range(3):
        h.copy_(dev)
    torch.cuda.synchronize()
    res[f"d2h_{name}_gbs"] = 3 * n / (time.perf_counter() - t0) / 1e9
cr = torch.cuda.cudart()
ptr = src.ctypes.data
t0 = time.perf_counter()
rc = cr.cudaHostRegister(ptr, n, 0)
res["host_register_s"] = time.perf_counter() - t0
res["host_register_rc"] = int(rc) if not isinstance(rc, tuple) else [int(x) for x in rc]
reg = torch.from_numpy(src.view(np.int16))
t0 = time.perf_counter()
for _ in range(3):
    dev.copy_(reg, non_blocking=True)
torch.cuda.synchronize()
res["h2d_registered_gbs"] = 3 * n / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter()
cr.cudaHostUnregister(ptr)
res["host_unregister_s"] = time.perf_counter() - t0
fresh = np.empty(n // 2, dtype=np.uint16)
t0 = time.perf_counter()
fresh[:] = 0
res["first_touch_fill_s"] = time.perf_counter() - t0
print(json.dumps(res))
