"""Pins of the oracle's randomized pieces (modification (2), P:359-362,
Appendix A): the counter-based Gaussian generator, the RSVD step,
the TT-RSVD fallback rule, and Table 1's I_QTT_r."""

import json
import math
import os

import numpy as np
import pytest

import oracle as O
from oracle import rng
from oracle.qtt import rsvd_step
from paper_2301_13339_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def test_generator_is_standard_normal():
    z = rng.omega(123, 4, np.arange(1 << 17), 16)
    assert abs(z.mean()) < 5e-3 and abs(z.var() - 1.0) < 5e-3
    # Kolmogorov-Smirnov distance to N(0,1) on 2^21 draws
    x = np.sort(z.reshape(-1))
    cdf = 0.5 * (1.0 + np.vectorize(math.erf)(x[::64] / math.sqrt(2.0)))
    emp = (np.arange(x.size)[::64] + 1) / x.size
    assert np.max(np.abs(cdf - emp)) < 2e-3
    # columns, steps and seeds are decorrelated
    c = np.corrcoef(z[:, :4].T)
    assert np.max(np.abs(c - np.eye(4))) < 1e-2
    z2 = rng.omega(123, 5, np.arange(1 << 17), 2)
    z3 = rng.omega(124, 4, np.arange(1 << 17), 2)
    assert abs(np.corrcoef(z[:, 0], z2[:, 0])[0, 1]) < 1e-2
    assert abs(np.corrcoef(z[:, 0], z3[:, 0])[0, 1]) < 1e-2
    # deterministic (counter-based): same counter, same value
    np.testing.assert_array_equal(rng.omega(123, 4, np.arange(5, 9), 16), z[5:9])


def test_rsvd_exact_on_low_rank():
    """rank(A) <= k: range(A Omega) = range(A) almost surely, so the RSVD
    reproduces A (Appendix A)."""
    r = np.random.default_rng(1)
    A = r.standard_normal((40, 7)) @ r.standard_normal((7, 300))
    U, s, Vh = rsvd_step(A, 8, 5, 99, 3)
    np.testing.assert_allclose((U * s) @ Vh, A, atol=1e-11 * np.linalg.norm(A))
    np.testing.assert_allclose(s[:7], np.linalg.svd(A, compute_uv=False)[:7], rtol=1e-12)


def test_rsvd_error_bound():
    """Eq. rsvd_error: ||A - A~|| <= (1 + 11 sqrt(k+p) sqrt(min(m,n)))
    sigma_{k+1} with probability >= 1 - 6 p^-p; after truncating to k
    singular values at most sigma_{k+1} more."""
    r = np.random.default_rng(2)
    k, p = 10, 5
    for t in range(20):
        Ua, _ = np.linalg.qr(r.standard_normal((100, 80)))
        Va, _ = np.linalg.qr(r.standard_normal((80, 80)))
        sig = 0.8 ** np.arange(80)
        A = (Ua * sig) @ Va.T
        U, s, Vh = rsvd_step(A, k, p, 1000 + t, 1)
        err = np.linalg.norm(A - (U[:, :k] * s[:k]) @ Vh[:k], 2)
        assert err <= (1 + 11 * math.sqrt(k + p) * math.sqrt(80)) * sig[k] + sig[k]


def test_tt_rsvd_fallback_and_low_rank():
    """min(m_k, n_k) <= R_max + p at every step -> the max-rank TT-SVD itself
    (P:366-367); exactly low-rank data -> the same ranks and reconstruction."""
    v = synth.random_signal((1 << 10,), 3)
    a = O.tt_svd(v, 1e-3, 10, 1e-10)
    b = O.tt_svd(v, 1e-3, 10, 1e-10, rsvd=(12, 5))      # R + p = 22 >= 2 r everywhere
    assert O.ranks_of(a) == O.ranks_of(b)
    np.testing.assert_allclose(O.full(a), O.full(b), atol=1e-12 * np.linalg.norm(v))
    # exactly rank-3 data, R = 3, p = 1: the 4-column sketch spans the range,
    # and the randomized branch is taken wherever min(m, n) = 6 > R + p = 4
    x = synth.random_signal((128, 128), 4, "lowrank")
    v = O.to_qtt(x, "interleaved")
    a = O.tt_svd(v, 1e-8, 3, 1e-10)
    b, info = O.tt_svd(v, 1e-8, 3, 1e-10, rsvd=(1, 5), return_info=True)
    assert sum(min(sh) > 4 for sh in info["unfolding_shapes"]) >= 5
    assert O.ranks_of(a) == O.ranks_of(b)
    np.testing.assert_allclose(O.full(b), v, atol=1e-9 * np.linalg.norm(v))


def _fft_conv(f, g, shift, scale):
    D = f.ndim
    gs = np.roll(g, tuple(-s for s in shift[::-1]), axis=tuple(range(D)))
    return scale * np.real(np.fft.ifftn(np.fft.fftn(f) * np.fft.fftn(gs)))


@pytest.mark.parametrize("num,K,key", [(1, 20, "example1_K20"), (2, 20, "example2_K20"), (3, 10, "example3_K10")])
def test_tt_rsvd_table1_paper_examples(num, K, key):
    """Table 1 I_QTT_r: R_max = 10, Rhat_max = 15, p = 5 (reading
    N2), eps = 1e-3 (as I_QTT0).  The randomised subspace loses accuracy
    against the max-rank TT-SVD exactly as printed (Example 1: 0.0101 vs
    0.0102); with p = 10 the same pipeline gives 0.0023 (outside the band)."""
    gold = GOLD["table1_E2_rsvd"][key]
    ex = synth.paper_example(num, K, noisy=True, seed=0)
    cl = synth.paper_example(num, K, noisy=False)
    sl = (slice(0, ex["N"]),) * ex["D"]
    ref = _fft_conv(cl["f"], cl["g"], ex["shift"], ex["scale"])[sl]
    lay = "1d" if ex["D"] == 1 else "concat"
    iq = O.conv_pipeline(ex["f"], ex["g"], lay, (1e-3, 10, 1e-10), (1e-3, 15, 1e-10), ex["shift"],
                         ex["scale"], rsvd=(5, 11, 12))[sl]
    e = np.linalg.norm(iq - ref) / np.linalg.norm(ref)
    assert 0.5 * gold <= e <= 2.0 * gold
