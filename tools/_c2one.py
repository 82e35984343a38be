import sys, torch
sys.path.insert(0, '.')
from paper_1705_08743_b200 import BoolMatrix, engines, workloads, _native
_native.lib().smx_set_graphs(0)
cfg = workloads.CONFIGS["c2_bool_warshall"]
(t,) = workloads.make_inputs(cfg, 4096)
m = BoolMatrix.from_numpy(t)
for _ in range(2):
    engines.bool_closure_bits(m); torch.cuda.synchronize()
