"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py
times (C3 4096^2, C4 16384^2, C5 the whole batch of 64 2048^2 images with a
shared kernel), at EVERY eps BASELINE.json lists for them, against the
oracle's result on the same seeded inputs as written by
tools/make_golden_fullsize.py (calls only oracle/):

  * identical ranks of F, G, their QTT-FFTs, the rounded product and the
    output (batch entry 0 through the report; every C5 image through the
    handle API);
  * the WHOLE output of every image through block fingerprints
    (tests/fingerprint.py: per 2^16-element block (2^18 at C4) its norm and
    two seeded projections), each block within 1e-9 of its norm (north
    star rel-L2 <= 1e-9);
  * every case is T2-gradable (the oracle's 1e-14 input-perturbation probe
    keeps all ranks and moves the output by <= 1e-11; recorded by the
    generator)."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from paper_2301_13339_b200 import qtt as Q
from paper_2301_13339_b200 import synth

from fingerprint import compare, fingerprint
from gpu_util import stream, ws

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(cfg):
    path = os.path.join(GOLD, f"fullsize_{cfg}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tools/make_golden_fullsize.py)")
    g = json.load(open(path))
    fp = np.load(os.path.join(GOLD, f"fullsize_{cfg}_fp.npz"))
    return g, fp


CASES = [("c3", 0), ("c3", 1), ("c5", 0), ("c5", 1), ("c5", 2), ("c4", 0)]


def test_golden_cases_are_gradable():
    """CPU check of the recorded T2 probe: every golden case keeps its ranks
    and moves by <= 1e-11 under 1e-14 input noise."""
    seen = 0
    for cfg in ("c3", "c4", "c5"):
        path = os.path.join(GOLD, f"fullsize_{cfg}.json")
        if not os.path.exists(path):
            continue
        g = json.load(open(path))
        for run in g["runs"]:
            assert run["probe"]["gradable"], (cfg, run["eps"], run["index"], run["probe"])
            assert run["min_margin"] > 0
            seen += 1
    assert seen > 0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,ei", CASES)
def test_fullsize_config_matches_oracle(cfg, ei):
    gold, fps = _gold(cfg)
    p = synth.problem(cfg)
    eps = gold["eps"][ei]
    runs = {r["index"]: r for r in gold["runs"] if r["eps"] == eps}
    n = 1 << p["d"]
    batch = p["batch"]
    g = synth.kernel(p["D"], p["b"], synth.CONFIGS[cfg]["w"])
    dev = torch.device("cuda", 0)
    fd = torch.empty(batch * n, dtype=torch.float64, device=dev)
    for i in range(batch):
        f = synth.signal(cfg, index=i)
        sha = hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest()
        assert sha == runs[i]["sha256_f"]
        fd[i * n:(i + 1) * n] = torch.from_numpy(np.ascontiguousarray(f).reshape(-1)).to(dev)
        del f
    assert hashlib.sha256(np.ascontiguousarray(g).tobytes()).hexdigest() == runs[0]["sha256_g"]
    gd = torch.from_numpy(np.ascontiguousarray(g).reshape(-1)).to(dev)
    shp = Q.shape(p["D"], [p["b"], p["b"]], p["layout"], batch, n, 0, n)
    dec = Q.trunc(eps, gold["caps"][0], gold["cluster_tol"])
    fft = Q.trunc(eps, gold["caps"][1], gold["cluster_tol"])
    nb = Q.qtt_workspace_bytes(shp, dec, fft)
    w = ws(nb)
    yd = torch.empty_like(fd)
    rep = Q.qtt_conv_full(fd.data_ptr(), gd.data_ptr(), yd.data_ptr(), shp, dec, fft, p["shift"], p["scale"],
                          w.data_ptr(), nb, stream(), report=True)
    torch.cuda.synchronize()
    assert rep["status_bits"] & 3 == 0
    r0 = runs[0]["ranks"]
    for key, st in (("ranks_f", "F"), ("ranks_g", "G"), ("ranks_fh", "Fh"), ("ranks_gh", "Gh"),
                    ("ranks_z", "Z"), ("ranks_out", "Y")):
        assert rep[key] == r0[st], (key, rep[key], r0[st])
    worst, est = 0.0, 0.0
    for i in range(batch):
        y = yd[i * n:(i + 1) * n].cpu().numpy()
        ok, wv, ev = compare(fingerprint(y), fps[f"eps{eps:g}_img{i}"])
        worst, est = max(worst, wv), max(est, ev)
        assert ok, (cfg, eps, i, wv)
    print(f"{cfg} eps={eps:g}: worst block deviation {worst:.2e}, est. rel-L2 {est:.2e}, "
          f"min margin {rep['min_margin']:.2e}")
    if batch > 1:
        # ranks of every image through the handle API (same kernels)
        del w, yd
        torch.cuda.empty_cache()
        w2 = ws(nb)
        tf = Q.qtt_decompose(fd.data_ptr(), shp, dec, w2.data_ptr(), nb, stream(), ws_owner=w2)
        shp1 = Q.shape(p["D"], [p["b"], p["b"]], p["layout"], 1)
        nb1 = Q.qtt_workspace_bytes(shp1, dec, fft)
        w3 = ws(nb1)
        tg = Q.qtt_decompose(gd.data_ptr(), shp1, dec, w3.data_ptr(), nb1, stream(), ws_owner=w3)
        w4 = ws(nb)
        ty = Q.qtt_convolve(tf, tg, fft, p["shift"], p["scale"], w4.data_ptr(), nb, stream(), ws_owner=w4)
        for i in range(batch):
            assert tf.ranks(i) == runs[i]["ranks"]["F"], i
            assert ty.ranks(i) == runs[i]["ranks"]["Y"], i
