"""Per-phase cycle counts of the small Hermitian eigensolver behind every
truncation (qtt_debug_eigh; TridSmem.tph: tridiagonalisation, eigenvalues,
eigenvector candidates, cluster re-orthogonalisation, back-transformation),
on graded PSD matrices shaped like the cut Grams K = M GR M^H, with the
agreement against LAPACK.  GPU only:
    python tools/eig_timing.py [n ...]
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2301_13339_b200 import qtt as Q  # noqa: E402

PHASES = ("tridiag", "eigenvalues", "vectors", "mgs", "backtransform")


def graded(n, seed, decades=8.0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    U, _ = np.linalg.qr(X)
    lam = np.logspace(0, -decades, n)
    A = (U * lam) @ U.conj().T
    return 0.5 * (A + A.conj().T)


def run(A, nvec, w20=False, reps=20, warm=False):
    n = A.shape[0]
    a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    U = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
    sw = torch.zeros(16, dtype=torch.int32, device="cuda")
    mode = ((64 + nvec) if warm else (2 + nvec)) | (256 if w20 else 0)
    Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(),
                     torch.cuda.current_stream().cuda_stream, mode=mode, reps=reps)
    torch.cuda.synchronize()
    u = U.cpu().numpy().view(np.complex128).reshape(n, n).T
    return lam.cpu().numpy(), u, sw.cpu().numpy()


def main(ns):
    Q.lib()
    for n in ns:
        for w20 in ((False, True) if n <= 16 else (True,)):
            A = graded(n, n)
            nvec = min(8, n)
            for _ in range(2):       # warm
                lg, ug, sw = run(A, nvec, w20)
            if "--warm" in sys.argv:
                _, _, sw2 = run(A, nvec, w20, warm=True)
                print(f"   second vector pass: {dict(zip(PHASES[2:], sw2[4:7].tolist()))}")
            lw = np.linalg.eigvalsh(A)[::-1]
            el = np.max(np.abs(lg - lw)) / np.abs(lw[0])
            res = np.linalg.norm(A @ ug[:, :nvec] - ug[:, :nvec] * lg[:nvec]) / np.linalg.norm(A)
            orth = np.linalg.norm(ug[:, :nvec].conj().T @ ug[:, :nvec] - np.eye(nvec))
            cyc = dict(zip(PHASES, sw[2:7].tolist()))
            if os.environ.get("QTT_LIB"):
                cyc["tridiag_steps"] = sw[7:12].tolist()
            print(f"n={n:2d} width={'20' if w20 else '16/32'} cycles {cyc} total {sum(sw[2:7])} "
                  f"| lam err {el:.1e} resid {res:.1e} orth {orth:.1e} fallbacks {sw[1]}", flush=True)


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:] if x.isdigit()] or [8, 12, 16, 20])
