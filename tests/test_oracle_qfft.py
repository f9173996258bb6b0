"""Pins for the oracle's QTT-FFT / QTT-iFFT, centering, Hadamard and rounding:
numpy.fft (library routine), closed-form DFTs, Parseval, the per-stage
partial-DFT invariant, exact element-wise products, lossless rounding.
"""

import numpy as np
import pytest

import oracle as O
from paper_2301_13339_b200 import synth

BIG = 10 ** 9


def _tt(v, eps=0.0, r=BIG):
    return O.tt_svd(v, eps, r)


@pytest.mark.parametrize("d", [3, 8, 12])
def test_qfft_1d_matches_numpy_fft(d):
    v = synth.random_signal((1 << d,), seed=d)
    ax = O.axes_descriptor(1, [d], "1d")
    Fh = O.qfft(_tt(v), ax, [d], 0.0, BIG)
    X = np.fft.fft(v)            # unnormalised, omega = e^{-2 pi i/N}
    assert np.linalg.norm(O.full(Fh) - X) <= 1e-13 * np.linalg.norm(X)


@pytest.mark.parametrize("layout", ["interleaved", "concat"])
def test_qfft_2d_matches_numpy_fft2_transposed(layout):
    # per-axis DFT; after the core reversal the x-frequency bits sit in the
    # y slots (F8): the QTT result is the layout of fft2(img).T
    b = 5
    img = synth.random_signal((1 << b, 1 << b), seed=2)
    ax = O.axes_descriptor(2, [b, b], layout)
    Fh = O.qfft(_tt(O.to_qtt(img, layout)), ax, [b, b], 0.0, BIG)
    X = np.fft.fft2(img)                        # X[ky, kx]
    got = O.from_qtt(O.full(Fh), img.shape, layout)
    assert np.linalg.norm(got - X.T) <= 1e-13 * np.linalg.norm(X)


def test_dft_closed_forms():
    d = 10
    n = 1 << d
    ax = O.axes_descriptor(1, [d], "1d")
    delta = np.zeros(n)
    delta[0] = 1.0
    Fh = O.qfft(_tt(delta, 1e-14), ax, [d], 1e-14, BIG)
    assert max(O.ranks_of(Fh)) == 1
    np.testing.assert_allclose(O.full(Fh), np.ones(n), atol=1e-13)
    Fh = O.qfft(_tt(np.ones(n), 1e-14), ax, [d], 1e-14, BIG)
    want = np.zeros(n)
    want[0] = n
    np.testing.assert_allclose(O.full(Fh), want, atol=1e-10)
    # DFT(e^{2 pi i k0 j/n}) = n delta_{k0}: the complex input enters as cores
    # built from the rank-1 factorisation of the exponential
    k0 = 37
    cores = [np.array([1.0, np.exp(2j * np.pi * k0 * (1 << k) / n)]).reshape(1, 2, 1)
             for k in range(d)]
    Fh = O.qfft(cores, ax, [d], 1e-14, BIG)
    want = np.zeros(n, complex)
    want[k0] = n
    np.testing.assert_allclose(O.full(Fh), want, atol=1e-9)


def test_parseval_exact_and_truncated():
    d = 12
    v = synth.random_signal((1 << d,), seed=4, kind="smooth")
    ax = O.axes_descriptor(1, [d], "1d")
    n2 = (1 << d) * np.dot(v, v)
    Fh = O.qfft(_tt(v), ax, [d], 0.0, BIG)
    e = O.full(Fh)
    assert abs(np.vdot(e, e).real - n2) <= 1e-13 * n2
    # with truncation every cut is an orthogonal projection: energy only
    # drops, by at most (d/2) eps^2 (reading Q29)
    for eps in (1e-2, 1e-4):
        Fh = O.qfft(_tt(v, 1e-12), ax, [d], eps, BIG)
        e = O.full(Fh)
        deficit = 1.0 - np.vdot(e, e).real / n2
        assert -1e-12 <= deficit <= (d / 2) * eps * eps
        X = np.fft.fft(v)
        assert np.linalg.norm(e - X) <= (2.0 / 3.0) * d * eps * np.linalg.norm(X)


def test_per_stage_partial_dft_invariant():
    # after s stages the tensor holds, for every j_low (low d-s bits), the
    # 2^s-point DFT of x(j_low + 2^{d-s} j_high) over j_high, with frequency
    # bit m at position d+1-m (radix-2 DIF)
    d = 8
    rng = np.random.default_rng(9)
    x = rng.standard_normal(1 << d) + 1j * rng.standard_normal(1 << d)
    # exact complex QTT of x (eps = 0) from real/imag TT-SVDs summed in TT form
    cr = O.tt_svd(x.real, 0.0, BIG)
    ci = O.tt_svd(x.imag, 0.0, BIG)
    cores = []
    for k in range(d):
        a, b = cr[k].astype(complex), ci[k] * (1j if k == 0 else 1.0)
        if k == 0:
            c = np.concatenate([a, b], axis=2)
        elif k == d - 1:
            c = np.concatenate([a, b], axis=0)
        else:
            c = np.zeros((a.shape[0] + b.shape[0], 2, a.shape[2] + b.shape[2]), complex)
            c[:a.shape[0], :, :a.shape[2]] = a
            c[a.shape[0]:, :, a.shape[2]:] = b
        cores.append(c)
    assert np.allclose(O.full(cores), x, atol=1e-12)
    ax = O.axes_descriptor(1, [d], "1d")
    for s in range(1, d + 1):
        T = O.full(O.qfft(cores, ax, [d], 0.0, BIG, stages=s))
        nlow = 1 << (d - s)
        for jl in range(0, nlow, max(1, nlow // 4)):
            seq = x[jl + nlow * np.arange(1 << s)]
            X = np.fft.fft(seq)
            for al in range(1 << s):
                pos = jl + sum(((al >> (m - 1)) & 1) << (d - m) for m in range(1, s + 1))
                assert abs(T[pos] - X[al]) <= 1e-11 * np.abs(X).max()


@pytest.mark.parametrize("layout", ["1d", "interleaved", "concat"])
def test_qifft_roundtrip(layout):
    if layout == "1d":
        v = synth.random_signal((1 << 10,), seed=1)
        ax, bits = O.axes_descriptor(1, [10], "1d"), [10]
    else:
        img = synth.random_signal((32, 32), seed=1)
        v = O.to_qtt(img, layout)
        ax, bits = O.axes_descriptor(2, [5, 5], layout), [5, 5]
    Fh = O.qfft(_tt(v), ax, bits, 0.0, BIG)
    Y = O.qifft(Fh, ax, bits, 0.0, BIG)
    back = O.full(Y)
    assert np.linalg.norm(back - v) <= 1e-13 * np.linalg.norm(v)


def test_center_is_dft_shift_theorem():
    # DFT of g_{(k + c) mod n} = e^{+2 pi i c alpha / n} DFT(g)   (O3)
    d = 9
    n = 1 << d
    g = synth.random_signal((n,), seed=8)
    ax = O.axes_descriptor(1, [d], "1d")
    Gh = O.qfft(_tt(g), ax, [d], 0.0, BIG)
    for c in (n // 2, 37, (n // 2 - 2) // 2):
        got = O.full(O.center(Gh, ax, [d], (c,)))
        want = np.fft.fft(np.roll(g, -c))
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_hadamard_elementwise_and_rank_product():
    rng = np.random.default_rng(3)
    rf = [1, 2, 3, 2, 1]
    rg = [1, 3, 2, 2, 1]
    F = [rng.standard_normal((rf[k], 2, rf[k + 1])) + 1j * rng.standard_normal((rf[k], 2, rf[k + 1])) for k in range(4)]
    G = [rng.standard_normal((rg[k], 2, rg[k + 1])) for k in range(4)]
    Z = O.hadamard(F, G)
    np.testing.assert_allclose(O.full(Z), O.full(F) * O.full(G), rtol=1e-13, atol=1e-13)
    assert O.ranks_of(Z) == [a * b for a, b in zip(rf, rg)]


def test_round_lossless_within_caps_and_rank1_residual():
    v = synth.random_signal((1 << 10,), seed=6, kind="lowrank")
    C = [c.astype(complex) for c in _tt(v, 1e-12)]
    R = O.round_full(C, 1e-14, BIG)
    assert np.linalg.norm(O.full(R) - v) <= 1e-13 * np.linalg.norm(v)
    # Kronecker of a rank-2 tensor with itself rounds to the exact square
    s = np.sin(0.3 * np.arange(1 << 10))
    S = [c.astype(complex) for c in _tt(s, 1e-13)]
    Z = O.round_full(O.hadamard(S, S), 1e-12, BIG)
    assert max(O.ranks_of(Z)) == 3              # sin^2 = (1 - cos 2x)/2
    assert np.linalg.norm(O.full(Z) - s * s) <= 1e-11 * np.linalg.norm(s * s)
    # MaxRank(1) rounding of a rank-2 two-core tensor leaves sigma_2
    A = np.array([[3.0, 0.0], [0.0, 1.0]])
    C = [c.astype(complex) for c in O.tt_svd(A.reshape(-1, order="F"), 0.0, BIG)]
    R = O.round_full(C, 0.0, 1)
    assert np.linalg.norm(O.full(R) - A.reshape(-1, order="F")) == pytest.approx(1.0, rel=1e-13)
