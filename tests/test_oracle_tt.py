"""Pins for the oracle's TT-SVD (Alg. 1 + mod (1)), rank rule and Full (Alg. 3).

Each test checks the oracle against something other than itself: closed-form
ranks, the paper's printed ranks and storage counts, exact reconstruction,
the Lemma 1 shapes, the eps error bound, brute force on tiny inputs.
"""

import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2301_13339_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))
BIG = 10 ** 9


# --------------------------------------------------------------------- layout

def test_qtt_pack_matches_bit_map():
    # V(i_1..i_K) = v(sum_k i_k 2^{k-1}); SPEC-style example
    v = np.array([10.0, 11.0, 12.0, 13.0])
    C = O.tt_svd(v, 0.0, BIG)
    assert O.element(C, 1)[0] == pytest.approx(11.0)     # i_1 = 1, i_2 = 0
    assert O.element(C, 2)[0] == pytest.approx(12.0)     # i_1 = 0, i_2 = 1


@pytest.mark.parametrize("layout", ["interleaved", "concat"])
def test_layout_roundtrip_and_bits(layout):
    b = 4
    img = np.arange(1 << (2 * b), dtype=float).reshape(1 << b, 1 << b)   # img[iy, ix]
    v = O.to_qtt(img, layout)
    np.testing.assert_array_equal(O.from_qtt(v, img.shape, layout), img)
    axes = O.axes_descriptor(2, [b, b], layout)
    rng = np.random.default_rng(0)
    for q in rng.integers(0, 1 << (2 * b), 50):
        ix = sum(((q >> p) & 1) << (t - 1) for p, (a, t) in enumerate(axes) if a == 0)
        iy = sum(((q >> p) & 1) << (t - 1) for p, (a, t) in enumerate(axes) if a == 1)
        assert v[q] == img[iy, ix]


# ------------------------------------------------------------------ rank rule

def test_rank_rule_eps_rank_definition():
    # rank_tau: minimal r with sum_{i>r} lam_i <= tau^2
    lam = np.array([16.0, 4.0, 1.0, 0.25, 0.0625])
    assert O.rank_rule(lam, 0.0625, BIG, 0.0) == 4     # T(4) = .0625 <= tau^2 (inclusive)
    assert O.rank_rule(lam, 0.06, BIG, 0.0) == 5
    assert O.rank_rule(lam, 0.3125, BIG, 0.0) == 3
    assert O.rank_rule(lam, 1.0e9, BIG, 0.0) == 1      # minimal rank is 1
    assert O.rank_rule(lam, 0.0, 2, 0.0) == 2          # max-rank cap
    assert O.rank_rule(np.zeros(4), 0.0, 3, 0.0) == 1  # zero input -> rank 1 (Q26)


def test_rank_rule_cluster_moves_cut_out_of_degenerate_pair():
    lam = np.array([9.0, 4.0, 4.0, 1.0, 1e-3])
    # plain rule (cluster test disabled) cuts between the equal pair (r = 2)
    assert O.rank_rule(lam, 5.5, BIG, -1.0) == 2
    # tolerance-bound cut moves up to the end of the cluster if the cap allows
    assert O.rank_rule(lam, 5.5, BIG, 1e-10) == 3
    # cap-bound cut moves down to the cluster start
    assert O.rank_rule(lam, 0.0, 2, 1e-10) == 1
    # non-degenerate neighbours are untouched
    assert O.rank_rule(np.array([9.0, 4.0, 3.9, 1.0]), 0.0, 2, 1e-10) == 2


# ---------------------------------------------------------- TT-SVD and Full

@pytest.mark.parametrize("d", [2, 5, 9, 13])
def test_exact_reconstruction_eps0_1d(d):
    v = synth.random_signal((1 << d,), seed=d)
    C = O.tt_svd(v, 0.0, BIG)
    assert np.linalg.norm(O.full(C) - v) <= 1e-13 * np.linalg.norm(v)
    # max unfolding rank of a generic tensor = min(2^k, 2^{d-k})
    assert O.ranks_of(C) == [1] + [min(2 ** k, 2 ** (d - k)) for k in range(1, d)] + [1]


@pytest.mark.parametrize("layout", ["interleaved", "concat"])
def test_exact_reconstruction_eps0_2d(layout):
    img = synth.random_signal((64, 64), seed=7)
    v = O.to_qtt(img, layout)
    C = O.tt_svd(v, 0.0, BIG)
    back = O.from_qtt(O.full(C), img.shape, layout)
    assert np.linalg.norm(back - img) <= 1e-13 * np.linalg.norm(img)


def test_closed_form_ranks_1d():
    d = 12
    j = np.arange(1 << d)
    # a^j = prod_k a^{i_k 2^{k-1}} is rank 1 at every cut
    assert max(O.ranks_of(O.tt_svd(0.999 ** j, 1e-12, BIG))) == 1
    assert max(O.ranks_of(O.tt_svd(np.full(1 << d, 3.0), 1e-12, BIG))) == 1
    # sin(w j + phi): every unfolding has rank 2
    r = O.ranks_of(O.tt_svd(np.sin(0.37 * j + 0.2), 1e-12, BIG))
    assert r[1:-1] == [2] * (d - 1)
    r = O.ranks_of(O.tt_svd(np.cos(0.011 * j), 1e-12, BIG))
    assert r[1:-1] == [2] * (d - 1)


def test_closed_form_ranks_2d_interleaved():
    b = 5
    x = np.arange(1 << b) / 32.0
    X, Y = np.meshgrid(x, x)
    r = O.ranks_of(O.tt_svd(O.to_qtt(np.exp(0.7 * X + 1.3 * Y), "interleaved"), 1e-12, BIG))
    assert max(r) == 1
    f = np.sin(3 * X + 0.1) * np.sin(5 * Y + 0.2)
    r = O.ranks_of(O.tt_svd(O.to_qtt(f, "interleaved"), 1e-12, BIG))
    # product of two rank-2 factors on interleaved bits: 2, 4, 4, ..., 4, 2
    assert r[1:-1] == [2] + [4] * (2 * b - 3) + [2]


def test_reconstruction_error_bound_when_no_cap_binds():
    # ||A - A~||_F <= eps ||A||_F (P:262-266 with tau of P:282, reading Q1)
    v = synth.random_signal((1 << 14,), seed=3, kind="smooth")
    for eps in (1e-2, 1e-4, 1e-8):
        C = O.tt_svd(v, eps, BIG)
        err = np.linalg.norm(O.full(C) - v)
        assert err <= eps * np.linalg.norm(v) * (1 + 1e-9)


def test_lemma1_unfolding_shapes():
    # Lemma 1: m_k = 2 r_{k-1} <= 2 R_max, n_k = 2^{K-k}
    d, R = 14, 10
    v = synth.random_signal((1 << d,), seed=11)
    C, info = O.tt_svd(v, 1e-3, R, return_info=True)
    r = O.ranks_of(C)
    for k, (m_k, n_k) in enumerate(info["unfolding_shapes"], start=1):
        assert m_k == 2 * r[k - 1] <= 2 * R
        assert n_k == 2 ** (d - k)


@pytest.mark.parametrize("d", [16, 20])
def test_storage_count_tables_3_and_5(d):
    # Tables 3/5, N_el formula P:709: noisy data with
    # R_max = 10 gives the staircase 2,4,8,10,...,10,8,4,2
    v = synth.random_signal((1 << d,), seed=d)
    C = O.tt_svd(v, 1e-3, 10)
    assert O.ranks_of(C) == [1, 2, 4, 8] + [10] * (d - 7) + [8, 4, 2, 1]
    want = GOLD["storage_rmax10"]["K_to_Nel_1d"][str(d)]
    assert O.storage_count(C) == want == 488 + 200 * (d - 8)
    assert GOLD["storage_rmax10"]["K_to_Nel_2d"][str(d // 2)] == want


def test_paper_max_ranks_example_1_and_2():
    # max TT-rank of the noise-free signals at eps = 1e-10,
    # K = 20.  Pins tau = eps ||A|| / sqrt(d-1), LSB-first bits
    # and the padded midpoint layout (readings Q1, Q7, F5).
    for num, key in ((1, "example1_K20_eps1e-10"), (2, "example2_K20_eps1e-10")):
        ex = synth.paper_example(num, 20)
        C = O.tt_svd(ex["f"], 1e-10, BIG)
        assert max(O.ranks_of(C)) == GOLD["max_tt_rank"][key]["value"]


def test_paper_max_rank_example_3_concat_layout():
    # 2D TT-rank 26 at K = 10 (d = 20); reproduces with concatenated
    # x-first bits (reading Q8, F6)
    ex = synth.paper_example(3, 10)
    C = O.tt_svd(O.to_qtt(ex["f"], "concat"), 1e-10, BIG)
    assert max(O.ranks_of(C)) == GOLD["max_tt_rank"]["example3_K10_eps1e-10"]["value"]


def test_full_matches_brute_force_contraction():
    # Alg. 3 vs the definition a(i) = A1[i1] ... AK[iK], random cores
    rng = np.random.default_rng(5)
    ranks = [1, 2, 3, 4, 3, 2, 1]
    cores = [rng.standard_normal((ranks[k], 2, ranks[k + 1])) for k in range(6)]
    f = O.full(cores)
    for q in range(64):
        m = np.eye(1)
        for k in range(6):
            m = m @ cores[k][:, (q >> k) & 1, :]
        assert f[q] == pytest.approx(m[0, 0], rel=1e-13, abs=1e-13)
    np.testing.assert_allclose(O.element(cores, np.arange(64)), f, rtol=1e-13, atol=1e-13)


def test_maxrank1_residual_is_sigma2():
    # rank-2 matrix as a 2-core QTT (d = 2): MaxRank(1) leaves sigma_2
    A = np.array([[3.0, 0.0], [0.0, 1.0]])
    v = A.reshape(-1, order="F")
    C = O.tt_svd(v, 0.0, 1)
    assert np.linalg.norm(O.full(C) - v) == pytest.approx(1.0, rel=1e-14)


def test_synth_blocks_reproduce_the_global_arrays():
    """Shard-wise input generation (multi-GPU bench) = slices of the global
    signal / kernel (same draws, same arithmetic)."""
    from paper_2301_13339_b200 import synth
    full = synth.signal("c2")
    clean = synth.signal("c2", noisy=False)
    cm = np.abs(clean).max()
    for (x0, nx, y0, ny) in [(0, 512, 0, 256), (0, 512, 256, 256), (256, 256, 256, 256), (128, 64, 300, 17)]:
        blk = synth.noisy_block("c2", 0, x0, nx, y0, ny, cm, row_chunk=100)
        np.testing.assert_allclose(blk, full[y0:y0 + ny, x0:x0 + nx], rtol=0, atol=1e-12)
    g = synth.kernel(2, 9, 60.0)
    np.testing.assert_allclose(synth.kernel_block(2, 9, 60.0, 256, 256, 0, 256), g[0:256, 256:512],
                               rtol=1e-14, atol=0)
    g1 = synth.kernel(1, 12, 40.0)
    np.testing.assert_allclose(synth.kernel_block(1, 12, 40.0, 1024, 1024), g1[1024:2048], rtol=1e-14)


# --------------------------------------------------------------- N3 drop-off
def test_dropoff_rule_cases():
    """Modification (3): keep sigma_1..sigma_k at the first
    relative drop sigma_{k+1}/sigma_k < delta (the rule sees lam = sigma^2)."""
    sig = np.array([1.0, 0.5, 0.004, 0.003])
    assert O.rank_rule_dropoff(sig ** 2, 0.02, 100, 1e-10) == 2        # 0.004/0.5 < 0.02
    assert O.rank_rule_dropoff(sig ** 2, 0.6, 100, 1e-10) == 1         # 0.5/1 < 0.6 first
    assert O.rank_rule_dropoff(sig ** 2, 0.001, 100, 1e-10) == 4       # no drop: all kept
    # no drop: the floor sigma_k >= 1e-7 sigma_1 decides (0.5^k >= 1e-7 for k <= 23)
    geo = 0.5 ** np.arange(40)
    assert O.rank_rule_dropoff(geo ** 2, 0.1, 100, 1e-10) == 24
    # capacity cap, and a cap inside a cluster moves down to the cluster start
    assert O.rank_rule_dropoff(geo ** 2, 0.1, 5, 1e-10) == 5
    assert O.rank_rule_dropoff(np.array([2.0, 1.0, 1.0, 1.0, 0.5]) ** 2, 0.1, 2, 1e-10) == 1
    assert O.rank_rule_dropoff(np.zeros(4), 0.1, 5, 1e-10) == 1


def test_dropoff_tt_svd_exact_low_rank():
    """An exactly rank-3 QTT (sum of three separable exponentials) has a drop
    of ~1e-16 after sigma_3 at every cut: the drop-off TT-SVD finds ranks
    <= 3 and reconstructs to rounding."""
    b = 7
    x = np.linspace(-1, 1, 1 << b, endpoint=False)
    X, Y = np.meshgrid(x, x)
    f = np.exp(0.7 * X + 0.2 * Y) + np.exp(-0.4 * X + 0.9 * Y) + np.exp(0.1 * X - 1.3 * Y)
    v = O.to_qtt(f, "interleaved")
    C = O.tt_svd(v, 0.0, 100, 1e-10, 1e-6)
    assert max(O.ranks_of(C)) <= 3
    assert np.linalg.norm(O.full(C) - v) <= 1e-12 * np.linalg.norm(v)


@pytest.mark.parametrize("num,K,key,lo,hi", [(1, 20, "example1_K20", 0.4, 2.5), (2, 20, "example2_K20", 0.7, 1.4),
                                             (3, 10, "example3_K10", 0.4, 2.5)])
def test_dropoff_table1_paper_examples(num, K, key, lo, hi):
    """Table 1 I_delta with the printed delta, uncapped, same delta
    in the TT-SVD and the QTT-FFT: Example 2 lands on the printed
    0.0068; the single-realisation Examples 1/3 within a factor 2.5."""
    gold = GOLD["table1_E2_dropoff"][key]
    ex = synth.paper_example(num, K, noisy=True, seed=0)
    cl = synth.paper_example(num, K, noisy=False)
    sl = (slice(0, ex["N"]),) * ex["D"]
    ref = _fft_conv(cl["f"], cl["g"], ex["shift"], ex["scale"])[sl]
    lay = "1d" if ex["D"] == 1 else "concat"
    tr = (0.0, 10 ** 6, 1e-10, gold["delta"])
    iq = O.conv_pipeline(ex["f"], ex["g"], lay, tr, tr, ex["shift"], ex["scale"])[sl]
    e = np.linalg.norm(iq - ref) / np.linalg.norm(ref)
    assert lo * gold["I_delta"] <= e <= hi * gold["I_delta"]


def _fft_conv(f, g, shift, scale):
    D = f.ndim
    gs = np.roll(g, tuple(-s for s in shift[::-1]), axis=tuple(range(D)))
    return scale * np.real(np.fft.ifftn(np.fft.fftn(f) * np.fft.fftn(gs)))
