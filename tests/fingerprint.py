"""Whole-array fingerprints of a full-size output (test infrastructure; no
method arithmetic).

A float64 array y of 2^d elements is cut into blocks of B = 2^16 elements
(2^18 at d >= 26).  Per block it keeps the L2 norm and two projections onto
fixed seeded N(0, 1) vectors r1, r2 of length B.  For a GPU result y' = y + e
a projection moves by <r, e_b> ~ N(0, ||e_b||^2): a block whose error is
above 1e-9 ||y_b|| fails the check with high probability, wherever in the
array the error sits (sampling 4096 positions could miss
an error confined to one expansion super-chunk).
"""

import numpy as np

SEED = 20260101


def block_size(n_el):
    return 1 << 18 if n_el >= (1 << 26) else 1 << 16


def _probes(B):
    rng = np.random.Generator(np.random.PCG64(SEED))
    return rng.standard_normal((B, 2))


def fingerprint(y):
    """(nblk, 3) array: per-block [||y_b||, <y_b, r1>, <y_b, r2>]."""
    y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
    B = block_size(y.size)
    Y = y.reshape(-1, B)
    out = np.empty((Y.shape[0], 3))
    out[:, 0] = np.linalg.norm(Y, axis=1)
    out[:, 1:] = Y @ _probes(B)
    return out


def compare(got, want, rel=1e-9):
    """Per-block check |d norm_b| <= rel ||y_b|| and |d proj_b| <= rel ||y_b||;
    returns (ok, worst ratio, estimated global rel-L2)."""
    got, want = np.asarray(got), np.asarray(want)
    scale = np.maximum(want[:, 0], 1e-300)
    dev = np.abs(got - want) / scale[:, None]
    est = float(np.sqrt(np.sum((got[:, 1:] - want[:, 1:]) ** 2) / 2.0) / np.sqrt(np.sum(want[:, 0] ** 2)))
    worst = float(dev.max())
    return worst <= rel, worst, est
