"""The paper's cap Rhat_max = 15: the
large-capacity transform variant (compact cores of rank <= 16 in the
workspace, 32-wide eigensolver) against the oracle, forward and inverse."""

import numpy as np
import pytest

import oracle as O
from paper_2301_13339_b200 import synth

from gpu_util import gpu_full, gpu_transform, gpu_tt_from_cores

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name,make,layout,eps", [
    ("1d_ex1_K16", lambda: synth.paper_example(1, 16, noisy=True)["f"], "1d", 1e-3),
    ("2d_concat_ex3_K8", lambda: synth.paper_example(3, 8, noisy=True)["f"], "concat", 1e-3),
    ("1d_noise_d14", lambda: synth.random_signal((1 << 14,), 61), "1d", 1e-3),
])
def test_transform_rhat15_parity(name, make, layout, eps):
    x = make()
    lay = "1d" if x.ndim == 1 else layout
    if x.ndim == 1:
        ax, bits = O.axes_descriptor(1, [int(np.log2(x.size))], "1d"), [int(np.log2(x.size))]
    else:
        b = int(np.log2(x.shape[0]))
        ax, bits = O.axes_descriptor(2, [b, b], lay), [b, b]
    F = O.tt_svd(O.to_qtt(x, lay), eps, 10, 1e-10)
    Fh = O.qfft(F, ax, bits, eps, 15, 1e-10)
    assert max(O.ranks_of(Fh)) > 10                      # the large variant is exercised
    tf = gpu_tt_from_cores(F, x, layout, rcap=10)
    th = gpu_transform(tf, None, eps, 15)
    assert th.ranks() == O.ranks_of(Fh)
    assert rel(gpu_full(th, x, imag=True), O.from_qtt(O.full(Fh), x.shape, lay)) <= 1e-9
    # inverse from the oracle's forward cores (ranks up to 15)
    Y = O.qifft(Fh, ax, bits, eps, 15, 1e-10)
    ti = gpu_transform(gpu_tt_from_cores(Fh, x, layout, rcap=16), None, eps, 15, inverse=True)
    assert ti.ranks() == O.ranks_of(Y)
    assert rel(gpu_full(ti, x, imag=True), O.from_qtt(O.full(Y), x.shape, lay)) <= 1e-9
