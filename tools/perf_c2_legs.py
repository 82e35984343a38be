"""Which leg binds the C2 closure (development aid; needs a library built
with SMX_EXTRA_NVCC_FLAGS=-DSMX_DEV_BOOL_SKIP): the blocked bit Warshall at
n = 4096 timed with legs of the schedule left out ($SMX_DEV_BOOL_SKIP mask:
1 = 3b, 2 = pivot, 4 = row panel, 8 = 3a; results are wrong in those runs)."""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, torch
sys.path.insert(0, '.')
from paper_1705_08743_b200 import BoolMatrix, engines, workloads
cfg = workloads.CONFIGS["c2_bool_warshall"]
(t,) = workloads.make_inputs(cfg, int(sys.argv[1]))
m = BoolMatrix.from_numpy(t)
for _ in range(3): engines.bool_closure_bits(m)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): engines.bool_closure_bits(m)
e.record(); torch.cuda.synchronize()
print(s.elapsed_time(e) / 20 * 1e3)
'''
n = sys.argv[1] if len(sys.argv) > 1 else "4096"
out = {"n": int(n)}
for mask, name in ((0, "all"), (1, "no_3b"), (14, "only_3b"), (2, "no_pivot"), (4, "no_row_panel"), (8, "no_3a"),
                   (9, "pivot_and_row_panel_only"), (13, "pivot_only"), (15, "nothing")):
    env = dict(os.environ, SMX_DEV_BOOL_SKIP=str(mask))
    r = subprocess.run([sys.executable, "-c", CHILD, n], env=env, capture_output=True, text=True)
    out[name + "_us"] = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
print(json.dumps(out))
