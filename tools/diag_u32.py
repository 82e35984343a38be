import sys, numpy as np, itertools
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import oracle
from paper_1705_08743_b200 import AntidistMatrix, DistMatrix, _native
from test_gpu_u32_packed import _graph
lib=_native.lib()
n=640; wmax=1<<31
rng=np.random.default_rng(n + (wmax & 0xFFFF))
t=_graph(rng,n,4.0/n,wmax,'anti')
want=oracle.semiring_close(t,32,'anti')
for p,b,l in itertools.product((0,1),(0,1),(0,1)):
    o=(lib.smx_set_fw_packed(p),lib.smx_set_bounded_fastpath(b),lib.smx_set_fw_lookahead(l))
    got=AntidistMatrix(n,n,32,t).transitive_closure().data
    print("packed",p,"bounded",b,"lookahead",l,"mismatch",int((got!=want).sum()),flush=True)
    lib.smx_set_fw_packed(o[0]);lib.smx_set_bounded_fastpath(o[1]);lib.smx_set_fw_lookahead(o[2])
# single products
for wm in (1000, 1<<31):
    a=_graph(rng,1024,0.3,wm,'anti')[:, :512].copy(); bb=_graph(rng,1024,0.3,wm,'anti')[:512].copy()
    for p in (0,1):
        o=lib.smx_set_fw_packed(p)
        got=(AntidistMatrix(1024,512,32,a)*AntidistMatrix(512,1024,32,bb)).data
        lib.smx_set_fw_packed(o)
        print("mul wmax",wm,"packed",p,"mismatch",int((got!=oracle.semiring_mul(a,bb,512,32,'anti')).sum()),flush=True)
