import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O
from paper_2301_13339_b200 import synth
from gpu_util import *
for name, x, lay in [("1d_noise_d16", synth.random_signal((1 << 16,), 41), "1d"),
                     ("1d_noise_d15", synth.random_signal((1 << 15,), 41), "1d"),
                     ("1d_noise_d14", synth.random_signal((1 << 14,), 41), "1d"),
                     ("2d_int_noise", synth.random_signal((256, 256), 43), "interleaved"),
                     ("2d_cat_noise", synth.random_signal((256, 256), 43), "concat")]:
    v = O.to_qtt(x, lay)
    d = int(np.log2(v.size))
    for p in (5, 2):
        ref, info = O.tt_svd(v, 1e-3, 10, 1e-10, rsvd=(p, 1234), return_info=True)
        tt = gpu_decompose_policy(x, lay, (1e-3, 10, 1e-10, None, (p, 1234)))
        g = O.to_qtt(gpu_full(tt, x), lay)
        fo = O.full(ref)
        act = [k + 1 for k, sh in enumerate(info["unfolding_shapes"]) if min(sh) > 10 + p]
        # per-prefix agreement: compare left-orthogonal subspaces step by step via partial contraction
        print(name, "p", p, "rsvd steps", act, "rel", "%.2e" % (np.linalg.norm(g - fo) / np.linalg.norm(fo)), flush=True)
