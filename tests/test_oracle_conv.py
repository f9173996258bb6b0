"""Pins for the oracle's end-to-end Alg. 2 pipeline: the convolution theorem
against brute-force O(n^2) periodic convolution (tiny n) and numpy FFT
convolution, and the paper's Table 1 errors on its own worked examples.
"""

import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2301_13339_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))
EXACT = (0.0, 10 ** 9, 1e-10)


def brute_1d(f, g, c, h):
    n = len(f)
    y = np.zeros(n)
    for j in range(n):
        for i in range(n):
            y[j] += f[i] * g[(j - i + c) % n]
    return h * y


def brute_2d(f, g, c, h):
    n = f.shape[0]
    y = np.zeros_like(f)
    for jy in range(n):
        for jx in range(n):
            s = 0.0
            for iy in range(n):
                for ix in range(n):
                    s += f[iy, ix] * g[(jy - iy + c[1]) % n, (jx - ix + c[0]) % n]
            y[jy, jx] = s
    return h * y


def fft_conv(f, g, c, h):
    """Periodic convolution via numpy.fft (library check)."""
    if f.ndim == 1:
        return h * np.real(np.fft.ifft(np.fft.fft(f) * np.fft.fft(np.roll(g, -c[0]))))
    gs = np.roll(np.roll(g, -c[1], axis=0), -c[0], axis=1)
    return h * np.real(np.fft.ifft2(np.fft.fft2(f) * np.fft.fft2(gs)))


@pytest.mark.parametrize("d,c", [(4, 8), (7, 64), (7, 37), (9, 0)])
def test_conv_theorem_1d_vs_brute_force(d, c):
    n = 1 << d
    f = synth.random_signal((n,), seed=d)
    g = synth.random_signal((n,), seed=d + 100)
    y = O.conv_pipeline(f, g, "1d", EXACT, EXACT, (c,), 0.5)
    want = brute_1d(f, g, c, 0.5)
    assert np.linalg.norm(y - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("layout", ["interleaved", "concat"])
@pytest.mark.parametrize("c", [(4, 4), (3, 5)])
def test_conv_theorem_2d_vs_brute_force(layout, c):
    n = 8
    f = synth.random_signal((n, n), seed=1)
    g = synth.random_signal((n, n), seed=2)
    y = O.conv_pipeline(f, g, layout, EXACT, EXACT, c, 0.25)
    want = brute_2d(f, g, c, 0.25)
    assert np.linalg.norm(y - want) <= 1e-12 * np.linalg.norm(want)


def test_conv_theorem_vs_numpy_fft_larger():
    f = synth.random_signal((1 << 12,), seed=3)
    g = synth.random_signal((1 << 12,), seed=4, kind="smooth")
    y = O.conv_pipeline(f, g, "1d", EXACT, EXACT, (1 << 11,), 1e-3)
    want = fft_conv(f, g, (1 << 11,), 1e-3)
    assert np.linalg.norm(y - want) <= 1e-12 * np.linalg.norm(want)
    f = synth.random_signal((64, 64), seed=5, kind="smooth")
    g = synth.random_signal((64, 64), seed=6, kind="smooth")
    y = O.conv_pipeline(f, g, "interleaved", EXACT, EXACT, (32, 32), 1e-3)
    want = fft_conv(f, g, (32, 32), 1e-3)
    assert np.linalg.norm(y - want) <= 1e-12 * np.linalg.norm(want)


def _e2(a, ref):
    # E_2; the 1/N^D of the norm cancels in the ratio
    return np.linalg.norm(a - ref) / np.linalg.norm(ref)


@pytest.mark.parametrize("num,K,key", [(1, 20, "example1_K20"), (2, 20, "example2_K20"),
                                       (3, 10, "example3_K10")])
def test_table1_errors_paper_examples(num, K, key):
    """Table 1.  E2(I_xi) (dense FFT of the noisy data) pins the
    harness: grid, padding, shift (N-1)/2, scale dx^D, kernel normalisation
    and sigma read as a standard deviation (F7).  E2(I_QTT0) (max-rank TT-SVD
    R_max = 10, QTT-FFT Rhat_max = 15, eps = 1e-3) pins the whole oracle
    pipeline on the paper's own worked example: it must land in the paper's
    regime (an order of magnitude below I_xi; paper 0.0028 / 0.0011 / 0.0151).
    """
    gold = GOLD["table1_E2"][key]
    ex = synth.paper_example(num, K, noisy=True, seed=0)
    cl = synth.paper_example(num, K, noisy=False)
    sl = (slice(0, ex["N"]),) * ex["D"]
    ref = fft_conv(cl["f"], cl["g"], ex["shift"], ex["scale"])[sl]
    ixi = fft_conv(ex["f"], ex["g"], ex["shift"], ex["scale"])[sl]
    assert _e2(ixi, ref) == pytest.approx(gold["I_xi"], rel=0.03)
    layout = "1d" if ex["D"] == 1 else "concat"
    iq = O.conv_pipeline(ex["f"], ex["g"], layout, (1e-3, 10, 1e-10), (1e-3, 15, 1e-10),
                         ex["shift"], ex["scale"])[sl]
    e = _e2(iq, ref)
    assert 0.25 * gold["I_QTT0"] <= e <= 2.0 * gold["I_QTT0"]
    assert e <= 0.5 * gold["I_xi"]
