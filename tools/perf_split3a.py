"""C4/C5 closure time with the look-ahead's 3a split (diagonal tile first,
pivot right behind it, the other columns on a second side stream) on and
off (development aid).  Prints JSON lines."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import _native, engines, workloads  # noqa: E402

lib = _native.lib()
for n in [int(x) for x in sys.argv[1:]] or [4096, 8192, 16384]:
    cfg = workloads.CONFIGS["c4_fw_u16" if n <= 8192 else "c5_fw_u16"]
    (x,) = workloads.make_inputs(cfg, n)
    src = torch.from_numpy(x).cuda()
    w = torch.empty_like(src)
    out = {"n": n}
    for rep, split in enumerate((0, 2, 0, 2)):
        old = lib.smx_set_fw_split_3a(split)
        try:
            def close():
                w.copy_(src)
                engines.lane_close_(w, n, 16, True)
            for _ in range(2):
                close()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            it = 3 if n >= 16384 else 10
            s.record()
            for _ in range(it):
                close()
            e.record()
            torch.cuda.synchronize()
            out[f"split{split}_ms_{rep // 2}"] = s.elapsed_time(e) / it
        finally:
            lib.smx_set_fw_split_3a(old)
    print(json.dumps(out), flush=True)
