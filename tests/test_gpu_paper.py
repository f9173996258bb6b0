"""NEXT row N1 on the GPU: the paper's own worked examples in
paper-faithful mode — midpoint grid with N = 2^{K-1} - 1 samples zero-padded
to 2^K per axis, kernel eq. sinc_kern1/2, linear
"same" convolution as the periodic one with shift (N-1)/2 followed by a crop
(reading Q10), 2D with concatenated bits (reading Q8, pinned by the
paper's rank 26).

Through the C ABI with caps (R_max, Rhat_max) = (10, 8) (reading Q4; the
paper's own caps (10, 15) are in test_gpu_rhat15.py):
identical ranks and rel-L2 <= 1e-9 against the oracle on the same inputs, and
the Table 1 quality regime: E2 of the QTT result against the exact
convolution of the clean signal well below E2 of the dense FFT of the noisy
data."""

import numpy as np
import pytest

import oracle as O
from paper_2301_13339_b200 import synth

from gpu_util import gpu_conv_full

pytestmark = pytest.mark.gpu

CAPS = ((1e-3, 10, 1e-10), (1e-3, 8, 1e-10))


def fft_conv(f, g, shift, scale):
    D = f.ndim
    gs = np.roll(g, tuple(-s for s in shift[::-1]), axis=tuple(range(D)))
    return scale * np.real(np.fft.ifftn(np.fft.fftn(f) * np.fft.fftn(gs)))


@pytest.mark.parametrize("num,K", [(1, 20), (2, 20), (3, 10)], ids=["ex1_K20", "ex2_K20", "ex3_K10"])
def test_paper_example_conv_on_gpu(num, K):
    ex = synth.paper_example(num, K, noisy=True, seed=0)
    cl = synth.paper_example(num, K, noisy=False)
    lay = "1d" if ex["D"] == 1 else "concat"
    dec, fft = CAPS
    y, rep = gpu_conv_full(ex["f"], ex["g"], lay, dec, fft, ex["shift"], ex["scale"])
    want, info = O.conv_pipeline(ex["f"], ex["g"], lay, dec, fft, ex["shift"], ex["scale"],
                                 return_info=True)
    assert rep["status_bits"] & 3 == 0
    assert rep["ranks_f"] == O.ranks_of(info["F"])
    assert rep["ranks_g"] == O.ranks_of(info["G"])
    assert rep["ranks_out"] == O.ranks_of(info["Y"])
    assert np.linalg.norm(y - want) <= 1e-9 * np.linalg.norm(want)
    # Table 1 regime on the cropped "same" output
    sl = (slice(0, ex["N"]),) * ex["D"]
    ref = fft_conv(cl["f"], cl["g"], ex["shift"], ex["scale"])[sl]
    e2 = lambda a: np.linalg.norm(a - ref) / np.linalg.norm(ref)   # noqa: E731
    e_qtt, e_xi = e2(y[sl]), e2(fft_conv(ex["f"], ex["g"], ex["shift"], ex["scale"])[sl])
    assert e_qtt <= 0.6 * e_xi
    assert abs(e_qtt - e2(want[sl])) <= 1e-6 * e_qtt
