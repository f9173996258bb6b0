"""Write the oracle's results on the FULL-size BASELINE configs C3, C4 and C5,
at EVERY eps BASELINE.json lists for them, for tests/test_gpu_fullsize.py:

  tests/golden/fullsize_<cfg>.json     ranks of F, G and the output of every
                                        image, SHA-256 of the inputs, the T2
                                        well-posedness probe
                                        and the minimum tail margin / gap of
                                        every run (oracle.margin_log)
  tests/golden/fullsize_<cfg>_fp.npz   whole-array fingerprints of every
                                        output image (tests/fingerprint.py:
                                        per-block norm + two seeded projections)

T2 probe: the pipeline is re-run on f (1 + 1e-14 N(0,1)) and g (1 + 1e-14
N(0,1)); the case is gradable at 1e-9 only if every rank (F, G, Fh, Gh, Z, Y)
is unchanged and the output moves by <= 1e-11 relative.

Calls only oracle/, the seeded input generator (paper_2301_13339_b200/
synth.py) and the fingerprint helper; nothing from the CUDA path.  Run on a
CPU host:
    python tools/make_golden_fullsize.py [c3 c4 c5] [--jobs N]
(C4 takes ~6 min per eps with its probe and ~12 GB of memory; C5 runs its
64 images x 3 eps x 2 (probe) pipelines over --jobs processes.)
"""

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from paper_2301_13339_b200 import synth  # noqa: E402
from fingerprint import fingerprint  # noqa: E402

STAGES = ("F", "G", "Fh", "Gh", "Z", "Y")


def perturb(x, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return x * (1.0 + 1e-14 * rng.standard_normal(x.shape))


def one(cfg, idx, eps, probe):
    p = synth.problem(cfg)
    c = synth.CONFIGS[cfg]
    dec = (eps, p["rmax"], p["cluster_tol"])
    fft = (eps, p["rhat"], p["cluster_tol"])
    g = synth.kernel(p["D"], p["b"], c["w"])
    f = synth.signal(cfg, index=idx)
    t0 = time.time()
    with O.margin_log() as ml:
        y, info = O.conv_pipeline(f, g, p["layout"], dec, fft, p["shift"], p["scale"], return_info=True)
    sec = time.time() - t0
    mg = np.array(ml) if ml else np.zeros((0, 2))
    rec = {"index": idx, "eps": eps,
           "sha256_f": hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest(),
           "sha256_g": hashlib.sha256(np.ascontiguousarray(g).tobytes()).hexdigest(),
           "ranks": {k: O.ranks_of(info[k]) for k in STAGES},
           "norm_y": float(np.linalg.norm(y)),
           "min_margin": float(mg[:, 0].min()) if len(mg) else None,
           "min_gap": float(mg[:, 1].min()) if len(mg) else None,
           "truncations": int(len(mg)),
           "oracle_seconds": round(sec, 2)}
    fp = fingerprint(y)
    if probe:
        y1, i1 = O.conv_pipeline(perturb(f, 7 + idx), perturb(g, 99), p["layout"], dec, fft, p["shift"],
                                 p["scale"], return_info=True)
        same = all(O.ranks_of(info[k]) == O.ranks_of(i1[k]) for k in STAGES)
        ch = float(np.linalg.norm(y1 - y) / np.linalg.norm(y))
        rec["probe"] = {"ranks_identical": bool(same), "rel_change": ch,
                        "gradable": bool(same and ch <= 1e-11)}
    return rec, fp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="*", default=["c3", "c5", "c4"])
    ap.add_argument("--jobs", type=int, default=max(1, (os.cpu_count() or 2) // 2))
    ap.add_argument("--no-probe", action="store_true")
    a = ap.parse_args()
    for cfg in a.cfgs:
        p = synth.problem(cfg)
        images = list(range(p["batch"]))
        out = {"_doc": "oracle result on the full-size config at every listed eps "
                       "(tools/make_golden_fullsize.py); fingerprints in fullsize_%s_fp.npz" % cfg,
               "config": cfg, "eps": p["eps"], "caps": [p["rmax"], p["rhat"]],
               "cluster_tol": p["cluster_tol"], "runs": []}
        fps = {}
        jobs = [(cfg, i, e, not a.no_probe) for e in p["eps"] for i in images]
        if len(jobs) > 1 and a.jobs > 1:
            os.environ.setdefault("OMP_NUM_THREADS", "2")
            with ProcessPoolExecutor(a.jobs) as ex:
                res = list(ex.map(one, *zip(*jobs)))
        else:
            res = [one(*j) for j in jobs]
        for (rec, fp) in res:
            out["runs"].append(rec)
            fps[f"eps{rec['eps']:g}_img{rec['index']}"] = fp
            pr = rec.get("probe", {})
            print(cfg, rec["eps"], rec["index"], "ranks Y", max(rec["ranks"]["Y"]), "margin",
                  f"{rec['min_margin']:.2e}", "gap", f"{rec['min_gap']:.2e}", "probe", pr, "s",
                  rec["oracle_seconds"], flush=True)
        gpath = os.path.join(ROOT, "tests", "golden", f"fullsize_{cfg}.json")
        with open(gpath, "w") as fh:
            json.dump(out, fh, indent=0)
        np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"fullsize_{cfg}_fp.npz"), **fps)
        print("wrote", gpath, flush=True)


if __name__ == "__main__":
    main()
