# stage-by-stage GPU vs oracle on the (16, 16)-caps 1D case (diagnostic)
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import oracle as O
from paper_2301_13339_b200 import synth
from gpu_util import gpu_decompose_policy, gpu_full, gpu_transform, gpu_tt_from_cores


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


f = synth.random_signal((1 << 14,), 91, kind="smooth") + 0.05 * synth.random_signal((1 << 14,), 92)
eps, R = 1e-6, 16
ax, bits = O.axes_descriptor(1, [14], "1d"), [14]
F = O.tt_svd(O.to_qtt(f, "1d"), eps, R, 1e-10)
tf = gpu_decompose_policy(f, "1d", (eps, R, 1e-10))
print("TT-SVD ranks equal", tf.ranks() == O.ranks_of(F), "rel", rel(gpu_full(tf, f), O.from_qtt(O.full(F), f.shape, "1d")))
Fh = O.qfft(F, ax, bits, eps, R, 1e-10)
th = gpu_transform(gpu_tt_from_cores(F, f, "1d", rcap=16), None, eps, R)
print("QFFT ranks equal", th.ranks() == O.ranks_of(Fh), "rel",
      rel(gpu_full(th, f, imag=True), O.from_qtt(O.full(Fh), f.shape, "1d")))
for Rin in (10, 12, 14):
    F2 = O.tt_svd(O.to_qtt(f, "1d"), eps, Rin, 1e-10)
    F2h = O.qfft(F2, ax, bits, eps, R, 1e-10)
    t2 = gpu_transform(gpu_tt_from_cores(F2, f, "1d", rcap=16), None, eps, R)
    print("QFFT in-rank", Rin, "ranks equal", t2.ranks() == O.ranks_of(F2h), "rel",
          rel(gpu_full(t2, f, imag=True), O.from_qtt(O.full(F2h), f.shape, "1d")))
Y = O.qifft(Fh, ax, bits, eps, R, 1e-10)
ti = gpu_transform(gpu_tt_from_cores(Fh, f, "1d", rcap=16), None, eps, R, inverse=True)
print("QiFFT ranks equal", ti.ranks() == O.ranks_of(Y), "rel",
      rel(gpu_full(ti, f, imag=True), O.from_qtt(O.full(Y), f.shape, "1d")))
