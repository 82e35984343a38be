import sys; sys.path.insert(0, '.')
import torch
from paper_1705_08743_b200 import BoolMatrix, workloads, _native, engines
lib = _native.lib(); lib.smx_set_graphs(0)
cfg = workloads.CONFIGS["c2_bool_warshall"]; (x,) = workloads.make_inputs(cfg)
m = BoolMatrix.from_numpy(x)
for _ in range(2):
    engines.bool_closure_bits(m)
torch.cuda.synchronize()
