"""NEXT row N3 on the GPU: the SV drop-off truncation
(modification (3); same delta in the TT-SVD and the QTT-FFT,
P:374-375) through the C ABI against the oracle's rank_rule_dropoff path:
identical ranks and rel-L2 <= 1e-9.  Ranks are capped at the kernels'
capacity (R_max = 10, Rhat = 8), in the oracle too."""

import numpy as np
import pytest

import oracle as O
from paper_2301_13339_b200 import synth

from gpu_util import gpu_conv_full, gpu_decompose_policy, gpu_full

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


CASES = [
    ("1d_smooth_d16", lambda: synth.random_signal((1 << 16,), 31, "smooth"), "1d", 0.02),
    ("2d_lowrank_d14", lambda: synth.random_signal((128, 128), 32, "lowrank"), "interleaved", 1e-4),
    ("2d_c2_signal", lambda: synth.signal("c2"), "interleaved", 0.02),
    ("2d_kernel_concat", lambda: synth.kernel(2, 8, 40.0), "concat", 0.05),
]


@pytest.mark.parametrize("name,make,layout,delta", CASES, ids=[c[0] for c in CASES])
def test_dropoff_decompose_parity(name, make, layout, delta):
    x = make()
    lay = "1d" if x.ndim == 1 else layout
    ref = O.tt_svd(O.to_qtt(x, lay), 0.0, 10, 1e-10, delta)
    tt = gpu_decompose_policy(x, layout, (0.0, 10, 1e-10, delta))
    assert tt.ranks() == O.ranks_of(ref)
    assert rel(gpu_full(tt, x), O.from_qtt(O.full(ref), x.shape, lay)) <= 1e-9


@pytest.mark.parametrize("num,K,delta", [(1, 20, 0.02), (2, 20, 0.01), (3, 10, 0.09)],
                         ids=["ex1_K20", "ex2_K20", "ex3_K10"])
def test_dropoff_conv_paper_examples(num, K, delta):
    ex = synth.paper_example(num, K, noisy=True, seed=0)
    lay = "1d" if ex["D"] == 1 else "concat"
    dec, fft = (0.0, 10, 1e-10, delta), (0.0, 8, 1e-10, delta)
    y, rep = gpu_conv_full(ex["f"], ex["g"], lay, dec, fft, ex["shift"], ex["scale"])
    want, info = O.conv_pipeline(ex["f"], ex["g"], lay, dec, fft, ex["shift"], ex["scale"],
                                 return_info=True)
    assert rep["status_bits"] & 3 == 0
    assert rep["ranks_f"] == O.ranks_of(info["F"])
    assert rep["ranks_out"] == O.ranks_of(info["Y"])
    assert rel(y, want) <= 1e-9
