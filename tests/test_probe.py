"""T2 well-posedness probe: a GPU-vs-oracle parity case is
only gradable at 1e-9 if the oracle itself is insensitive to rounding-level
perturbations of its input.  Each chained (end-to-end) parity case of
tests/test_gpu_parity.py is probed here: relative input noise of 1e-14 must
move the result by <= 1e-11 and leave every rank unchanged.  The one chained
case that fails the probe (forward -> inverse at eps = 1e-6 on a smooth
signal) is documented here and tested stage-isolated on the GPU instead."""

import numpy as np
import pytest

import oracle as O
from paper_2301_13339_b200 import synth


def _perturb(x, seed):
    rng = np.random.default_rng(seed)
    return x * (1.0 + 1e-14 * rng.standard_normal(x.shape))


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_configs_are_well_posed(cfg):
    p = synth.problem(cfg)
    f = synth.signal(cfg)
    g = synth.kernel(p["D"], p["b"], synth.CONFIGS[cfg]["w"])
    eps = p["eps"][0]
    dec, fft = (eps, p["rmax"], 1e-10), (eps, p["rhat"], 1e-10)
    y0, i0 = O.conv_pipeline(f, g, p["layout"], dec, fft, p["shift"], p["scale"], return_info=True)
    y1, i1 = O.conv_pipeline(_perturb(f, 1), g, p["layout"], dec, fft, p["shift"], p["scale"],
                             return_info=True)
    assert np.linalg.norm(y1 - y0) <= 1e-11 * np.linalg.norm(y0)
    for k in ("F", "G", "Fh", "Gh", "Z", "Y"):
        assert O.ranks_of(i0[k]) == O.ranks_of(i1[k])


def test_documented_ill_posed_chain():
    # forward -> inverse chain at eps = 1e-6, smooth d = 16 input: the cap
    # binds where the kept singular values are ~3e-5 sigma_1 and rounding
    # noise is amplified ~1e3x; parity of this chain is not gradable at 1e-9
    d = 16
    x = synth.random_signal((1 << d,), 11, "smooth")
    ax, bits = O.axes_descriptor(1, [d], "1d"), [d]

    def chain(v):
        h = O.qfft(O.tt_svd(v, 1e-6, 10, 1e-10), ax, bits, 1e-6, 8, 1e-10)
        return O.full(O.qifft(h, ax, bits, 1e-6, 8, 1e-10))

    i0, i1 = chain(x), chain(_perturb(x, 2))
    assert np.linalg.norm(i1 - i0) > 1e2 * 1e-14 * np.linalg.norm(i0)
