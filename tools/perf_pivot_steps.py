import ctypes, json, sys
sys.path.insert(0, '.')
import torch
from paper_1705_08743_b200 import _native, workloads, engines
lib = _native.lib()
cfg = workloads.CONFIGS["c4_fw_u16"]
(T,) = workloads.make_inputs(cfg, 8192)
src = torch.from_numpy(T).cuda()
w = src.clone()
engines.lane_close_(w, 8192, 16, True)   # a closed matrix: bounded tiles, as in later rounds
res = {}
for name, base in (("input", src), ("closed", w)):
    t = base[:1024].clone()
    for rep in range(3):
        lib.smx_fw_trace_arm(64)
        _native.check(lib.smx_fw_pivot(t.data_ptr(), 256, t.shape[1], 2, 0, _native.stream_ptr()), "pivot")
        torch.cuda.synchronize()
        ms = (ctypes.c_float * 64)(); cells = (ctypes.c_longlong * 64)()
        k = lib.smx_fw_trace_read(ms, cells, 64)
    res[name] = {f"step{-cells[i]-10}": ms[i] for i in range(k)}
print(json.dumps(res))
