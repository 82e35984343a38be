import sys, json, torch, time
sys.path.insert(0,'.')
from paper_1705_08743_b200 import engines, workloads
n=32768
cfg=workloads.CONFIGS["c5_mul_u16"]; a,b=workloads.make_inputs(cfg,n)
da=torch.from_numpy(a).cuda(); db=torch.from_numpy(b).cuda()
res={}
for groups in (1,2,4,8):
    g=n//groups
    def run():
        for r0 in range(0,n,g):
            engines.lane_mul(da[r0:r0+g], db, n, 16, True)
    run(); torch.cuda.synchronize()
    t0=time.perf_counter(); run(); torch.cuda.synchronize()
    res[groups]=(time.perf_counter()-t0)*1e3
print(json.dumps(res))
