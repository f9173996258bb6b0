import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O
from paper_2301_13339_b200 import synth, qtt as Q
from gpu_util import *
print(Q.build_info())
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300)
for name, x, lay, eps, r in [("1d10", synth.random_signal((1<<10,),1), "1d", 1e-3, 10),
                             ("1d16", synth.random_signal((1<<16,),3), "1d", 1e-3, 10),
                             ("2d14", synth.random_signal((128,128),5), "interleaved", 1e-3, 10)]:
    try:
        t=time.time()
        ref = O.tt_svd(O.to_qtt(x, "1d" if x.ndim==1 else lay), eps, r, 1e-10)
        tt = gpu_decompose(x, lay, eps, r)
        print(name, 'gpu ranks', tt.ranks()); print(name, 'ora ranks', O.ranks_of(ref))
        got = gpu_full(tt, x)
        want = O.from_qtt(O.full(ref), x.shape, "1d" if x.ndim==1 else lay)
        print(name, 'rel', rel(got, want), time.time()-t)
    except Exception as e:
        print(name, 'ERR', e)
