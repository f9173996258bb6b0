"""Expansion (Alg. 3) store paths: the staged 16-byte row stores of
k_expand_main for every layout, an output pointer that is only 8-byte aligned
(falls back to 8-byte stores), and a batch whose y_stride is odd — each
against the oracle's full() of the same cores."""

import numpy as np
import pytest
import torch

import oracle as O
from paper_2301_13339_b200 import qtt as Q
from paper_2301_13339_b200 import synth

from gpu_util import gpu_tt_from_cores, stream, ws

pytestmark = pytest.mark.gpu


def _oracle_full(F, x, layout):
    return O.from_qtt(np.real(O.full(F)), x.shape, layout)


@pytest.mark.parametrize("layout,shape", [("interleaved", (256, 256)), ("concat", (256, 256)),
                                          ("1d", (1 << 16,))])
@pytest.mark.parametrize("offset", [0, 1])
def test_expand_staged_stores(layout, shape, offset):
    x = synth.random_signal(shape, 5, kind="smooth")
    F = O.tt_svd(O.to_qtt(x, layout), 1e-6, 10, 1e-10)
    tt = gpu_tt_from_cores(F, x, layout, rcap=10)
    n = x.size
    buf = torch.full((n + 2,), float("nan"), dtype=torch.float64, device="cuda")
    w = ws(1 << 22)
    Q.qtt_to_full(tt, buf.data_ptr() + 8 * offset, w.data_ptr(), 1 << 22, stream())
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    want = _oracle_full(F, x, layout)
    assert np.isnan(got[:offset]).all() and np.isnan(got[offset + n:]).all()   # nothing outside y
    y = got[offset:offset + n].reshape(x.shape)
    assert np.linalg.norm(y - want) <= 1e-12 * np.linalg.norm(want)


def test_conv_batch_odd_y_stride():
    """qtt_conv_full with y_stride = n + 1 (every other batch entry 8-byte
    aligned only) against the aligned run."""
    b = 8
    n = 1 << (2 * b)
    f = np.stack([synth.random_signal((1 << b, 1 << b), 40 + i, kind="smooth") for i in range(2)])
    g = synth.random_signal((1 << b, 1 << b), 49, kind="smooth")
    fd = torch.from_numpy(f.reshape(-1)).cuda()
    gd = torch.from_numpy(g.reshape(-1)).cuda()
    dec, fft = Q.trunc(1e-6, 10), Q.trunc(1e-6, 8)
    outs = []
    for ys in (n, n + 1):
        shp = Q.shape(2, [b, b], "interleaved", 2, n, 0, ys)
        nb = Q.qtt_workspace_bytes(shp, dec, fft)
        w = ws(nb)
        y = torch.zeros(2 * ys, dtype=torch.float64, device="cuda")
        Q.qtt_conv_full(fd.data_ptr(), gd.data_ptr(), y.data_ptr(), shp, dec, fft, (128, 128), 1.0,
                        w.data_ptr(), nb, stream())
        torch.cuda.synchronize()
        yc = y.cpu().numpy()
        outs.append(np.stack([yc[i * ys:i * ys + n] for i in range(2)]))
    assert np.array_equal(outs[0], outs[1])
