"""Oracle: the counter-based Gaussian generator of the randomized SVD
(modification (2); Appendix A "Draw random matrix Omega_ij ~
N(0,1)").

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

The paper draws Omega with MATLAB's randn; for GPU/oracle parity both sides
implement the same counter-based generator (reading N2-rng):
  * a Philox-4x32 bijection with 10 rounds (Salmon et al., SC'11): per round
    (c0, c1, c2, c3) <- (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2), hi(M0 c0) ^ c3 ^ k1,
    lo(M0 c0)) with M0 = 0xD2511F53, M1 = 0xCD9E8D57, then the key is bumped
    by (0x9E3779B9, 0xBB67AE85);
  * two 53-bit uniforms u = ((w_a >> 5) 2^26 + (w_b >> 6) + 1/2) 2^-53 in
    (0, 1) from the four output words, and the Box-Muller pair
    z0 = sqrt(-2 ln u1) cos(2 pi u2), z1 = sqrt(-2 ln u1) sin(2 pi u2);
  * Omega_k[j, c] of TT-SVD step k: counter (j mod 2^32, j >> 32, k, c >> 1),
    key (seed mod 2^32, seed >> 32), value z_{c mod 2}.
Written with numpy uint64 arithmetic, vectorised over j only.
"""

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten rounds on uint64 arrays holding 32-bit values; returns 4 words."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & MASK for x in (c0, c1, c2, c3))
    k0, k1 = int(k0) & MASK, int(k1) & MASK
    for _ in range(10):
        p0 = c0 * np.uint64(M0)
        p1 = c2 * np.uint64(M1)
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK)
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
        k0 = (k0 + W0) & MASK
        k1 = (k1 + W1) & MASK
    return c0, c1, c2, c3


def _u53(wa, wb):
    a = (wa >> np.uint64(5)).astype(np.float64)
    b = (wb >> np.uint64(6)).astype(np.float64)
    return (a * 67108864.0 + b + 0.5) * (1.0 / 9007199254740992.0)


def omega(seed, k, j, ncols):
    """Omega_k[j, 0:ncols] for an integer array of rows j (float64 (len(j), ncols))."""
    j = np.asarray(j, dtype=np.uint64)
    out = np.empty((j.shape[0], ncols))
    for cp in range((ncols + 1) // 2):
        x0, x1, x2, x3 = philox4x32_10(j & np.uint64(MASK), j >> np.uint64(32),
                                       np.full(j.shape, k, np.uint64), np.full(j.shape, cp, np.uint64),
                                       seed & MASK, seed >> 32)
        u1, u2 = _u53(x0, x1), _u53(x2, x3)
        rad = np.sqrt(-2.0 * np.log(u1))
        out[:, 2 * cp] = rad * np.cos(2.0 * np.pi * u2)
        if 2 * cp + 1 < ncols:
            out[:, 2 * cp + 1] = rad * np.sin(2.0 * np.pi * u2)
    return out
