import sys; sys.path.insert(0,'.')
import torch
from paper_1705_08743_b200 import engines, workloads, _native
lib=_native.lib(); lib.smx_set_graphs(0)
cfg=workloads.CONFIGS["c5_fw_u16"]; (x,)=workloads.make_inputs(cfg, 32768)
w=torch.from_numpy(x).cuda()
engines.lane_close_(w, 32768, 16, True); torch.cuda.synchronize()
