import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O
from paper_2301_13339_b200 import synth
from gpu_util import *
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300)
for d, eps in [(16, 1e-6), (16, 1e-3), (12, 1e-6)]:
    x = synth.random_signal((1 << d,), 11, "smooth")
    ax, bits = O.axes_descriptor(1, [d], "1d"), [d]
    ref = O.tt_svd(x, eps, 10, 1e-10)
    refh = O.qfft(ref, ax, bits, eps, 8, 1e-10)
    refi = O.qifft(refh, ax, bits, eps, 8, 1e-10)
    # GPU forward on the oracle's TT-SVD cores
    t0 = gpu_tt_from_cores(ref, x, "1d")
    th = gpu_transform(t0, x, eps, 8)
    print(d, eps, 'fwd ranks eq', th.ranks()==O.ranks_of(refh), 'fwd rel', rel(gpu_full(th, x, imag=True), O.full(refh)))
    # GPU inverse on the oracle's forward cores
    t1 = gpu_tt_from_cores(refh, x, "1d")
    ti = gpu_transform(t1, x, eps, 8, inverse=True)
    print(d, eps, 'inv ranks eq', ti.ranks()==O.ranks_of(refi), 'inv rel', rel(gpu_full(ti, x, imag=True), O.full(refi)))
