"""Memory-safety and determinism evidence for the whole path (SURVEY §4.2 T4 /
T6).  compute-sanitizer is closed on this pool (runs under it left GPUs
needing a reset), so out-of-bounds writes are caught with guard bands
instead: the workspace is followed by a canary region, the output is
surrounded by NaN guards, the inputs are checked bit for bit afterwards.
T6: the same call twice gives bitwise identical outputs and ranks (the
per-CTA partial Grams are reduced in a fixed order, no floating-point
atomics)."""

import numpy as np
import pytest
import torch

from paper_2301_13339_b200 import qtt as Q
from paper_2301_13339_b200 import synth

from gpu_util import stream

pytestmark = pytest.mark.gpu

CASES = [
    ("c1", 1),
    ("c2", 1),
    ("c2_batch3", 3),
    ("2d_concat_d16", 1),
]


def _inputs(name, batch):
    if name.startswith("c1"):
        p = synth.problem("c1")
        f = np.stack([synth.signal("c1", index=i) for i in range(batch)])
        g = synth.kernel(1, p["b"], synth.CONFIGS["c1"]["w"])
        shp = Q.shape(1, [p["b"], 0], "1d", batch)
        return f, g, shp, p["shift"], p["scale"], p["eps"][0]
    if name.startswith("c2"):
        p = synth.problem("c2")
        f = np.stack([synth.signal("c2", index=i) for i in range(batch)])
        g = synth.kernel(2, p["b"], synth.CONFIGS["c2"]["w"])
        shp = Q.shape(2, [p["b"], p["b"]], "interleaved", batch)
        return f, g, shp, p["shift"], p["scale"], p["eps"][0]
    b = 8
    f = synth.random_signal((1 << b, 1 << b), 5, "smooth")[None]
    g = synth.kernel(2, b, 30.0)
    shp = Q.shape(2, [b, b], "concat", 1)
    return f, g, shp, (1 << (b - 1), 1 << (b - 1)), (2.0 / (1 << b)) ** 2, 1e-3


@pytest.mark.parametrize("name,batch", CASES, ids=[c[0] for c in CASES])
def test_guard_bands_and_determinism(name, batch):
    f, g, shp, shift, scale, eps = _inputs(name, batch)
    n = f[0].size
    dec, fft = Q.trunc(eps, 10), Q.trunc(eps, 8)
    nb = Q.qtt_workspace_bytes(shp, dec, fft)
    canary = 1 << 20
    ws = torch.empty(nb + canary + 256, dtype=torch.uint8, device="cuda")
    base = (ws.data_ptr() + 255) & ~255
    off = base - ws.data_ptr()
    ws[off + nb: off + nb + canary].fill_(0xA5)
    fd = torch.from_numpy(np.ascontiguousarray(f).reshape(-1)).cuda()
    gd = torch.from_numpy(np.ascontiguousarray(g).reshape(-1)).cuda()
    f0, g0 = fd.clone(), gd.clone()
    guard = 4096
    ybuf = torch.full((guard + batch * n + guard,), float("nan"), dtype=torch.float64, device="cuda")
    yd = ybuf[guard:guard + batch * n]
    outs, reps = [], []
    for _ in range(2):
        rep = Q.qtt_conv_full(fd.data_ptr(), gd.data_ptr(), yd.data_ptr(), shp, dec, fft, shift, scale, base, nb,
                              stream(), report=True)
        torch.cuda.synchronize()
        outs.append(yd.clone())
        reps.append(rep)
    # nothing written past the workspace, around y, or into the inputs
    assert bool((ws[off + nb: off + nb + canary] == 0xA5).all())
    assert bool(torch.isnan(ybuf[:guard]).all()) and bool(torch.isnan(ybuf[guard + batch * n:]).all())
    assert torch.equal(fd, f0) and torch.equal(gd, g0)
    assert bool(torch.isfinite(outs[0]).all())
    # T6: bitwise identical run to run
    assert torch.equal(outs[0], outs[1])
    for k in ("ranks_f", "ranks_g", "ranks_fh", "ranks_gh", "ranks_z", "ranks_out", "status_bits"):
        assert reps[0][k] == reps[1][k], k
    assert reps[0]["min_margin"] == reps[1]["min_margin"]
