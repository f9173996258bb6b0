"""The paper's own timing workloads on the GPU (PAPER.md
Tables 2 and 4, with the storage of Tables 3 and 5,
P:689-693 and P:846-850): Example 1 (1D) at K = 16..28 and Example 3 (2D,
concatenated bits) at K = 8..14, I_QTT0 = max-rank TT-SVD + capped QTT-FFT
convolution + Full at the paper's caps (R_max, Rhat_max) = (10, 15), eps =
1e-3 (Table 1's setting), paper-linear mode (zero padding, shift (N-1)/2).

Per workload: device time of one qtt_conv_full (inputs resident, CUDA events,
after warm-up), the storage of the signal's QTT (sum_k r_{k-1} 2 r_k, the
paper's Tables 3/5 quantity), the maximum output rank, and E2 of the cropped
result against the dense convolution of the clean signal.  The
paper's MATLAB times (hardware unstated) are printed beside as context.

    python tools/paper_tables.py [--out profiles/r01h_paper_tables.json]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2301_13339_b200 import qtt as Q  # noqa: E402
from paper_2301_13339_b200 import synth  # noqa: E402

PAPER_S = {(1, 16): 0.325, (1, 20): 0.653, (1, 24): 4.41, (1, 26): 17.75, (1, 28): 95.5,
           (3, 8): 0.2213, (3, 10): 0.9209, (3, 12): 8.6462, (3, 14): 147.8}
PAPER_STORAGE = {16: 2088, 20: 2888, 24: 3688, 26: 4088, 28: 4488}


def dense_conv(f, g, shift, scale, dev):
    D = f.ndim
    ft = torch.from_numpy(f).to(dev)
    gt = torch.roll(torch.from_numpy(g).to(dev), shifts=tuple(-s for s in shift[::-1]), dims=tuple(range(D)))
    dims = tuple(range(D))
    return (torch.fft.irfftn(torch.fft.rfftn(ft, dim=dims) * torch.fft.rfftn(gt, dim=dims), s=f.shape, dim=dims)
            * scale)


def run(num, K, dev, reps=3):
    ex = synth.paper_example(num, K, noisy=True, seed=0)
    cl = synth.paper_example(num, K, noisy=False)
    D = ex["D"]
    lay = "1d" if D == 1 else "concat"
    n = ex["f"].size
    fd = torch.from_numpy(np.ascontiguousarray(ex["f"]).reshape(-1)).to(dev)
    gd = torch.from_numpy(np.ascontiguousarray(ex["g"]).reshape(-1)).to(dev)
    yd = torch.empty(n, dtype=torch.float64, device=dev)
    shp = Q.shape(1, [K, 0], "1d") if D == 1 else Q.shape(2, [K, K], "concat")
    dec, fft = Q.trunc(1e-3, 10, 1e-10), Q.trunc(1e-3, 15, 1e-10)
    nb = Q.qtt_workspace_bytes(shp, dec, fft)
    ws = torch.empty(nb + 256, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream

    def step(report=False):
        return Q.qtt_conv_full(fd.data_ptr(), gd.data_ptr(), yd.data_ptr(), shp, dec, fft, ex["shift"],
                               ex["scale"], ws.data_ptr(), nb, st, report=report)
    rep = step(report=True)
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        step()
    ev1.record()
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1) / reps
    rf = rep["ranks_f"]
    storage = int(sum(rf[k] * 2 * rf[k + 1] for k in range(len(rf) - 1)))
    sl = (slice(0, ex["N"]),) * D
    ref = dense_conv(np.ascontiguousarray(cl["f"]), np.ascontiguousarray(cl["g"]), ex["shift"], ex["scale"], dev)
    y = yd.view(ex["f"].shape)
    e2 = float(torch.linalg.vector_norm(y[sl] - ref[sl]) / torch.linalg.vector_norm(ref[sl]))
    out = {"example": num, "K": K, "elements": n, "gpu_ms": ms, "paper_matlab_s": PAPER_S.get((num, K)),
           "storage_f": storage, "max_rank_f": max(rf), "max_rank_out": max(rep["ranks_out"]),
           "e2_vs_clean_conv": e2, "status_bits": rep["status_bits"]}
    if num == 1 and K in PAPER_STORAGE:
        out["paper_storage"] = PAPER_STORAGE[K]
    del fd, gd, yd, ws, ref
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    rows = []
    for num, K in [(1, 16), (1, 20), (1, 24), (1, 26), (1, 28), (3, 8), (3, 10), (3, 12), (3, 14)]:
        r = run(num, K, dev)
        rows.append(r)
        print(json.dumps(r), flush=True)
    if a.out:
        json.dump({"_doc": __doc__.split("\n\n")[0], "caps": [10, 15], "eps": 1e-3, "rows": rows},
                  open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
