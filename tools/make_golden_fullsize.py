"""Write tests/golden/fullsize_<cfg>.json: the float64 oracle's result on the
FULL-size BASELINE configs C3, C4 and C5 (C5: images 0, 29, 63 of the batch),
as identical-rank data (ranks of F, G and the output) and the output at 4096
seeded sample positions plus its full L2 norm, for tests/test_gpu_fullsize.py.

Calls only oracle/ and the seeded input generator (paper_2301_13339_b200/
synth.py); nothing from the CUDA path.  Run on a CPU host:
    python tools/make_golden_fullsize.py [c3 c4 c5]
(C4 takes several minutes and ~10 GB of memory.)
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2301_13339_b200 import synth  # noqa: E402

IMAGES = {"c3": [0], "c4": [0], "c5": [0, 29, 63]}
NSAMPLE = 4096


def sample_positions(n_el, seed):
    rng = np.random.default_rng(seed)
    q = rng.integers(0, n_el, NSAMPLE - 2, dtype=np.int64)
    return np.concatenate([[0, n_el - 1], q])


def main(cfgs):
    for cfg in cfgs:
        p = synth.problem(cfg)
        c = synth.CONFIGS[cfg]
        eps = p["eps"][0]
        dec = (eps, p["rmax"], p["cluster_tol"])
        fft = (eps, p["rhat"], p["cluster_tol"])
        g = synth.kernel(p["D"], p["b"], c["w"])
        out = {"_doc": "oracle result on the full-size config (tools/make_golden_fullsize.py); "
                       "output samples y.flat[idx] (row-major), full-array L2 norm",
               "config": cfg, "eps": eps, "caps": [p["rmax"], p["rhat"]], "cluster_tol": p["cluster_tol"],
               "images": []}
        for idx in IMAGES[cfg]:
            t0 = time.time()
            f = synth.signal(cfg, index=idx)
            y, info = O.conv_pipeline(f, g, p["layout"], dec, fft, p["shift"], p["scale"], return_info=True)
            pos = sample_positions(y.size, 1000 + idx)
            out["images"].append({
                "index": idx,
                "sha256_f": hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest(),
                "ranks_f": O.ranks_of(info["F"]), "ranks_g": O.ranks_of(info["G"]),
                "ranks_out": O.ranks_of(info["Y"]),
                "norm_y": float(np.linalg.norm(y)),
                "sample_idx": pos.tolist(), "sample_val": y.reshape(-1)[pos].tolist(),
                "oracle_seconds": round(time.time() - t0, 1)})
            print(cfg, idx, "ranks out", O.ranks_of(info["Y"])[:6], "s", round(time.time() - t0, 1), flush=True)
            del f, y, info
        path = os.path.join(ROOT, "tests", "golden", f"fullsize_{cfg}.json")
        with open(path, "w") as fh:
            json.dump(out, fh)
        print("wrote", path, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3", "c5", "c4"])
