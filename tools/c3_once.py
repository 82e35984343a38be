import sys; sys.path.insert(0, '.')
import torch
from paper_1705_08743_b200 import engines, workloads, _native
lib = _native.lib(); lib.smx_set_graphs(0)
cfg = workloads.CONFIGS["c3_mul_u16"]; a, b = workloads.make_inputs(cfg)
ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
res = torch.empty_like(ta)
for _ in range(2):
    engines.lane_mul(ta, tb, cfg.n, cfg.width, True, res)
torch.cuda.synchronize()
