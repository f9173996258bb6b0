"""NEXT row N2 on the GPU: the max-rank TT-RSVD
(modification (2); Appendix A) through the C ABI against
the oracle's tt_svd(..., rsvd=(p, seed)): the same counter-based Omega on both
sides (compared element-wise), identical ranks and rel-L2 <= 1e-9 of the
decompositions and of the end-to-end convolution."""

import numpy as np
import pytest
import torch

import oracle as O
from oracle import rng
from paper_2301_13339_b200 import qtt as Q
from paper_2301_13339_b200 import synth

from gpu_util import gpu_conv_full, gpu_decompose_policy, gpu_full, stream

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("seed,k,j0", [(0, 1, 0), (12345678901, 7, 1 << 33), (2 ** 63 + 5, 22, 99)])
def test_omega_matches_oracle(seed, k, j0):
    n, kp = 4096, 15
    out = torch.empty(n * kp, dtype=torch.float64, device="cuda")
    Q.qtt_debug_omega(seed, k, j0, n, kp, out.data_ptr(), stream())
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(n, kp)
    want = rng.omega(seed, k, np.arange(j0, j0 + n, dtype=np.uint64), kp)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-13)


CASES = [
    ("1d_noise_d16", lambda: synth.random_signal((1 << 16,), 41), "1d", 1e-3, 10, 5),
    ("1d_noise_d12_finisher", lambda: synth.random_signal((1 << 12,), 42), "1d", 1e-3, 10, 5),
    ("2d_c2_signal", lambda: synth.signal("c2"), "interleaved", 1e-3, 10, 5),
    ("2d_noise_p2", lambda: synth.random_signal((256, 256), 43), "interleaved", 1e-3, 10, 2),
    ("2d_smooth_concat", lambda: synth.random_signal((256, 256), 44, "smooth"), "concat", 1e-4, 8, 4),
]


@pytest.mark.parametrize("name,make,layout,eps,rmax,p", CASES, ids=[c[0] for c in CASES])
def test_rsvd_decompose_parity(name, make, layout, eps, rmax, p):
    x = make()
    lay = "1d" if x.ndim == 1 else layout
    seed = 1000 + len(name)
    ref, info = O.tt_svd(O.to_qtt(x, lay), eps, rmax, 1e-10, rsvd=(p, seed), return_info=True)
    assert any(min(sh) > rmax + p for sh in info["unfolding_shapes"])      # the randomized branch ran
    tt = gpu_decompose_policy(x, layout, (eps, rmax, 1e-10, None, (p, seed)))
    assert tt.ranks() == O.ranks_of(ref)
    assert rel(gpu_full(tt, x), O.from_qtt(O.full(ref), x.shape, lay)) <= 1e-9


@pytest.mark.parametrize("num,K", [(1, 20), (3, 10)], ids=["ex1_K20", "ex3_K10"])
def test_rsvd_conv_paper_examples(num, K):
    ex = synth.paper_example(num, K, noisy=True, seed=0)
    lay = "1d" if ex["D"] == 1 else "concat"
    seed = 77
    dec, fft = (1e-3, 10, 1e-10, None, (5, seed)), (1e-3, 8, 1e-10)
    y, rep = gpu_conv_full(ex["f"], ex["g"], lay, dec, fft, ex["shift"], ex["scale"])
    want, info = O.conv_pipeline(ex["f"], ex["g"], lay, (1e-3, 10, 1e-10), fft, ex["shift"], ex["scale"],
                                 return_info=True, rsvd=(5, seed, seed + 1))
    assert rep["ranks_f"] == O.ranks_of(info["F"])
    assert rep["ranks_g"] == O.ranks_of(info["G"])
    assert rep["ranks_out"] == O.ranks_of(info["Y"])
    assert rel(y, want) <= 1e-9
