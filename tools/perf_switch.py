"""A/B timing of one library switch on the u16 FW closure, same process and
GPU (development aid):

    python tools/perf_switch.py smx_set_fw_pivot_pairs 0 1 -- 4096 8192

Each setting is timed twice, interleaved (A B A B), 10 closures each (3 at
n >= 16384) after two warm-ups that record the replay graph.  JSON lines."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import _native, engines, workloads  # noqa: E402

argv = sys.argv[1:]
cut = argv.index("--") if "--" in argv else len(argv)
switch, values = argv[0], [int(v) for v in argv[1:cut]]
sizes = [int(x) for x in argv[cut + 1:]] or [4096, 8192]
lib = _native.lib()
setter = getattr(lib, switch)
for n in sizes:
    cfg = workloads.CONFIGS["c4_fw_u16" if n <= 8192 else "c5_fw_u16"]
    (x,) = workloads.make_inputs(cfg, n)
    src = torch.from_numpy(x).cuda()
    w = torch.empty_like(src)
    out = {"n": n, "switch": switch}
    for rep in range(2):
        for v in values:
            old = setter(v)
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
                out[f"v{v}_ms_{rep}"] = s.elapsed_time(e) / it
            finally:
                setter(old)
    print(json.dumps(out), flush=True)
