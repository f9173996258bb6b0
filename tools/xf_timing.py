"""Per-phase cycles of the QTT-FFT kernel k_transform (needs a diagnostic
build with -DQTT_XF_TIMING; CTA 0's clock64 totals are dumped into the tail
of its right-Gram scratch).  GPU only:
    python tools/xf_timing.py        # builds paper_2301_13339_b200/libqtt_xf.so
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
XF_LIB = os.path.join(ROOT, "paper_2301_13339_b200", "libqtt_xf.so")
if "QTT_LIB" not in os.environ:
    from paper_2301_13339_b200 import build as B
    if not os.environ.get("XF_NOBUILD"):
        B.build(out=XF_LIB, extra=["-DQTT_XF_TIMING"])
    os.environ["QTT_LIB"] = XF_LIB

import torch  # noqa: E402

from paper_2301_13339_b200 import qtt as Q  # noqa: E402
from paper_2301_13339_b200 import synth  # noqa: E402
from gpu_util import gpu_decompose, stream, ws  # noqa: E402

NAMES = ["GR chain (products)", "K formation", "eig values", "push", "GR write", "cut start", "rank", "vectors"]


def run(x, label, eps=1e-3, rhat=8):
    tt = gpu_decompose(x, "interleaved", eps, 10)
    fft = Q.trunc(eps, rhat)
    nb = 64 << 20
    w = ws(nb)
    Q.qtt_transform(tt, fft, 0, None, 1.0, w.data_ptr(), nb, stream(), ws_owner=w)
    torch.cuda.synchronize()
    raw = w.cpu().numpy().view(np.int64)
    d = int(np.log2(x.size))
    off = 0

    def take(nbytes):
        nonlocal off
        off = (off + 255) & ~255
        o = off
        off += nbytes
        return o

    take(d * 512 * 16)
    take(64 * 4)
    gr = take(30 * 400 * 16)
    base = (gr + (30 * 400 - 8) * 16) // 8
    cyc = raw[base:base + 8]
    cuts = d * (d - 1) // 2
    tot = cyc.sum()
    print(f"{label}: d={d} total {tot / 1.965e3:.0f} us = {tot / 1.965e3 / cuts:.2f} us per cut | " +
          " ".join(f"{n}={c / 1.965e3 / cuts:.2f}" for n, c in zip(NAMES, cyc)), flush=True)


if __name__ == "__main__":
    run(synth.signal("c2"), "F(c2)")
    run(synth.kernel(2, 9, 60.0), "G(c2 kernel)")
    run(synth.signal("c3"), "F(c3)", eps=1e-2)
