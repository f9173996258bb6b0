"""Oracle: QTT layout, the truncation rank rule, TT-SVD (Alg. 1 + max-rank
modification (1)) and Full (Alg. 3).

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.  Plain numpy float64,
written to be checked against PAPER.md by eye; no blocking, fusion or
reordering beyond what Alg. 1 / Alg. 3 state.
"""

import numpy as np


# ---------------------------------------------------------------------------
# QTT layout (readings Q7, Q8)
# ---------------------------------------------------------------------------

def axes_descriptor(D, bits, layout):
    """(axis, bit) for every QTT position p = 1..d (returned 0-based list).

    P:303 fixes 1D: i = sum_k i_k 2^{k-1}, LSB first (reading Q7).
    leaves the 2D mode order open (reading Q8): 'interleaved' puts x-bit t at
    position 2t-1 and y-bit t at 2t (x first); 'concat' puts all x-bits, then
    all y-bits.  `bit` is 1-based, LSB = 1.
    """
    if D == 1:
        return [(0, t) for t in range(1, bits[0] + 1)]
    bx, by = bits
    if layout == "interleaved":
        if bx != by:
            raise ValueError("interleaved layout needs a square grid")
        out = []
        for t in range(1, bx + 1):
            out.append((0, t))
            out.append((1, t))
        return out
    if layout == "concat":
        return [(0, t) for t in range(1, bx + 1)] + [(1, t) for t in range(1, by + 1)]
    raise ValueError(layout)


def to_qtt(x, layout="1d"):
    """Vector v in QTT order: v[sum_p i_p 2^{p-1}] = x at the grid point whose
    axis bits are the i_p.

    1D / concat: the array in memory (row-major image, x fastest) is already
    in QTT order.  Interleaved: position 2t-1 is x-bit t, 2t is y-bit t.
    """
    x = np.asarray(x)
    if layout in ("1d", "concat") or x.ndim == 1:
        return np.ascontiguousarray(x).reshape(-1)
    ny, nx = x.shape
    b = int(np.log2(nx))
    assert nx == ny == 1 << b
    # image[iy, ix] with iy = sum y_t 2^{t-1}; C-order axes (y_b..y_1, x_b..x_1)
    t = x.reshape([2] * (2 * b))
    # QTT index q = x1 + 2 y1 + 4 x2 + ...; as a C-order array its axes are
    # (y_b, x_b, y_{b-1}, x_{b-1}, ..., y_1, x_1)
    order = []
    for k in range(b):          # k = 0 is the most significant bit
        order.append(k)         # y_{b-k}
        order.append(b + k)     # x_{b-k}
    return np.ascontiguousarray(t.transpose(order)).reshape(-1)


def from_qtt(v, shape, layout="1d"):
    """Inverse of to_qtt."""
    v = np.asarray(v)
    if layout in ("1d", "concat") or len(shape) == 1:
        return v.reshape(shape)
    ny, nx = shape
    b = int(np.log2(nx))
    t = v.reshape([2] * (2 * b))          # axes (y_b, x_b, ..., y_1, x_1)
    inv = [2 * k for k in range(b)] + [2 * k + 1 for k in range(b)]
    return np.ascontiguousarray(t.transpose(inv)).reshape(shape)


# ---------------------------------------------------------------------------
# Rank rule: eps-rank + max-rank modification (1)
# + cluster rule (reading Q6 / SURVEY §8(c) O1 RANK)
# ---------------------------------------------------------------------------

def rank_rule(lam, tau2, rmax, cluster_tol):
    """RANK(lambda, tau^2, R, delta_c).

    lam: squared singular values, descending.  T(r) = sum_{i>r} lam_i is
    accumulated from the smallest value up.  r_tau = min{r >= 1 : T(r) <=
    tau^2} is rank_tau of P:286 (inclusive <=, reading Q2); r = min(r_tau, R)
    is modification (1) (reading Q3).  A cut inside a cluster of
    (numerically) equal values, lam_r - lam_{r+1} <= delta_c lam_r, is moved
    up to the end of the cluster when the tolerance allows it and the cap
    still holds, else down to its start (reading Q6; the gap is relative to
    lam_r, not lam_1 — with lam_1 every value below sqrt(delta_c) sigma_1 is
    one "cluster" and the paper's ranks 17/26 come out full,
    DESIGN.md §3 reading Q6').
    """
    lam = np.maximum(np.asarray(lam, dtype=np.float64), 0.0)
    m = lam.shape[0]
    if m == 0 or not lam[0] > 0.0:
        return 1
    tail = np.zeros(m + 1)                 # tail[r] = T(r), r = 0..m
    for r in range(m - 1, -1, -1):
        tail[r] = tail[r + 1] + lam[r]
    r_tau = m
    for r in range(1, m + 1):
        if tail[r] <= tau2:
            r_tau = r
            break
    r = min(r_tau, rmax)

    def cl(q):
        return q < m and lam[q - 1] > 0.0 and \
            (lam[q - 1] - lam[q]) <= cluster_tol * lam[q - 1]

    if cl(r):
        if r_tau <= rmax:
            rp = r + 1
            while cl(rp):
                rp += 1
            if rp <= rmax:
                _log_margin(lam, tail, tau2, r_tau, rmax, rp)
                return rp
        while r > 1 and cl(r):
            r -= 1
    _log_margin(lam, tail, tau2, r_tau, rmax, r)
    return r


# ---------------------------------------------------------------------------
# T2 well-posedness diagnostics.  Logging only: nothing here
# feeds back into a rank or a value.
# ---------------------------------------------------------------------------

_MARGIN_LOG = None


class margin_log:
    """Context manager: while active, every RANK decision appends
    (margin, gap) to the list it yields.  margin = distance of the deciding
    tail sum(s) from tau^2, relative to tau^2 — |T(r_tau) - tau^2| and
    |T(r_tau - 1) - tau^2| when eps decides (r_tau <= R), |T(R) - tau^2| when
    the cap does; gap = (lam_r - lam_{r+1}) / lam_1 at the returned r (inf
    when r = m).  SURVEY §4.2 T2 flags a cut when |T - tau^2| is within the
    Gram noise (~1e3 m eps_mach lam_1) or the gap within [0.1, 10] delta_c."""

    def __enter__(self):
        global _MARGIN_LOG
        self.prev, self.rows = _MARGIN_LOG, []
        _MARGIN_LOG = self.rows
        return self.rows

    def __exit__(self, *exc):
        global _MARGIN_LOG
        _MARGIN_LOG = self.prev
        return False


def _log_margin(lam, tail, tau2, r_tau, rmax, r):
    if _MARGIN_LOG is None or not tau2 > 0.0:
        return
    m = lam.shape[0]
    if r_tau <= rmax:
        mg = abs(tail[r_tau] - tau2)
        if r_tau > 1:
            mg = min(mg, abs(tail[r_tau - 1] - tau2))
    else:
        mg = abs(tail[rmax] - tau2)
    gap = (lam[r - 1] - lam[r]) / lam[0] if r < m else float("inf")
    _MARGIN_LOG.append((mg / tau2, gap))


def rank_rule_dropoff(lam, delta, rmax, cluster_tol):
    """SV drop-off rule, modification (3): "if sigma_{k+1} /
    sigma_k < delta ... truncate the singular values less than sigma_k", i.e.
    keep sigma_1..sigma_k for the FIRST k (from the top) with a relative drop;
    on lam = sigma^2 the test is lam_{k+1} < delta^2 lam_k.

    Readings (N3): without a drop above it, values below the
    floor sigma_k < 1e-7 sigma_1 (lam_k < 1e-14 lam_1) are discarded (the
    paper is silent; SPEC S:149 floors at 1e-14 sigma_1, which only an SVD of
    the unfolding resolves, not its Gram); the kernel capacity cap r <= R is
    applied last and, when it cuts inside a cluster (Q6'), the cut moves
    down to the cluster start as in RANK.
    """
    lam = np.maximum(np.asarray(lam, dtype=np.float64), 0.0)
    m = lam.shape[0]
    if m == 0 or not lam[0] > 0.0:
        return 1
    floor = 0
    for k in range(m):
        if lam[k] >= 1e-14 * lam[0]:
            floor = k + 1
    r_d = floor
    for k in range(1, m):
        if lam[k] < delta * delta * lam[k - 1]:
            r_d = min(k, floor)
            break
    r = min(r_d, rmax)

    def cl(q):
        return q < m and lam[q - 1] > 0.0 and \
            (lam[q - 1] - lam[q]) <= cluster_tol * lam[q - 1]

    if r < r_d:
        while r > 1 and cl(r):
            r -= 1
    return max(r, 1)


def choose_rank(lam, tau2, rmax, cluster_tol, delta=None):
    """RANK (modifications (1)) or, with delta given, the drop-off rule (3)."""
    if delta is None:
        return rank_rule(lam, tau2, rmax, cluster_tol)
    return rank_rule_dropoff(lam, delta, rmax, cluster_tol)


# ---------------------------------------------------------------------------
# Alg. 1 TT-SVD with modification (1)
# ---------------------------------------------------------------------------

def rsvd_step(A, k, p, seed, step):
    """Randomized SVD of Appendix A (Alg. "Solving the Fixed-Rank
    Problem" + Alg. "RSVD", [HMT11] Alg. 5.1): Omega (n x (k+p)) ~ N(0,1)
    (oracle.rng, counter = TT-SVD step), Y = A Omega, Q R = Y, B = Q^* A,
    U~ Sigma V^* = B, U = Q U~.  Returns (U, s, Vh) like numpy.linalg.svd."""
    from .rng import omega
    n = A.shape[1]
    Om = omega(seed, step, np.arange(n), k + p)
    Y = A @ Om
    Q, _ = np.linalg.qr(Y)
    B = Q.conj().T @ A
    Ut, s, Vh = np.linalg.svd(B, full_matrices=False)
    return Q @ Ut, s, Vh


def tt_svd(v, eps, rmax, cluster_tol=1e-10, delta=None, return_info=False, rsvd=None):
    """Max-rank TT-SVD of a 2x...x2 tensor given as its QTT-ordered vector.

    tau = eps ||A||_F / sqrt(d-1) (P:282 with M-1 read as d-1, reading Q1).
    Step k: A^{k} = reshape(A, [2 r_{k-1}, |A|/(2 r_{k-1})]) (column-major,
    P:234/P:248), truncated SVD with ||E||_F <= tau and r_k <= R_max,
    core_k = reshape(U, [r_{k-1}, 2, r_k]), A := Sigma V^* (P:285-288);
    core_d := A.  With `delta` the truncation is modification (3)
    (SV drop-off, rank_rule_dropoff) instead of eps / R_max.  With
    rsvd = (p, seed) the SVD of step k is the randomized SVD with k = R_max
    and oversampling p (modification (2)), except when
    min(m_k, n_k) <= R_max + p, where it reverts to the SVD.
    """
    v = np.asarray(v, dtype=np.float64).reshape(-1)
    n = v.shape[0]
    d = int(round(np.log2(n)))
    if (1 << d) != n or d < 2:
        raise ValueError("length must be 2^d with d >= 2")
    norm2 = float(np.dot(v, v))
    tau2 = eps * eps * norm2 / (d - 1)
    cores = []
    shapes = []
    r_prev = 1
    W = v
    for k in range(1, d):
        M = np.reshape(W, (2 * r_prev, -1), order="F")
        shapes.append(M.shape)
        if rsvd is not None and min(M.shape) > rmax + rsvd[0]:
            U, s, Vt = rsvd_step(M, rmax, rsvd[0], rsvd[1], k)
        else:
            U, s, Vt = np.linalg.svd(M, full_matrices=False)
        r = choose_rank(s * s, tau2, rmax, cluster_tol, delta)
        cores.append(np.reshape(U[:, :r], (r_prev, 2, r), order="F"))
        W = s[:r, None] * Vt[:r, :]
        r_prev = r
    cores.append(np.reshape(W, (r_prev, 2, 1), order="F"))
    if return_info:
        return cores, {"unfolding_shapes": shapes, "tau2": tau2, "norm2": norm2}
    return cores


def ranks_of(cores):
    """r_0 .. r_d."""
    return [cores[0].shape[0]] + [c.shape[2] for c in cores]


def storage_count(cores):
    """N_el = sum_k r_{k-1} M_k r_k."""
    return int(sum(c.size for c in cores))


# ---------------------------------------------------------------------------
# Alg. 3 Full and single elements
# ---------------------------------------------------------------------------

def full(cores):
    """A = core_1; for k = 2..K: A = reshape(A, [|A|/r_{k-1}, r_{k-1}]) @
    reshape(core_k, [r_{k-1}, 2 r_k]); return the QTT-ordered vector."""
    r1 = cores[0].shape[2]
    A = np.reshape(cores[0], (2, r1), order="F")
    for k in range(1, len(cores)):
        c = cores[k]
        rk_1, _, rk = c.shape
        A = np.reshape(A, (A.size // rk_1, rk_1), order="F") @ \
            np.reshape(c, (rk_1, 2 * rk), order="F")
    return np.reshape(A, (-1,), order="F")


def element(cores, q):
    """a(i_1..i_K) = A^(1)_{i_1} ... A^(K)_{i_K} at QTT indices q
    (scalar or 1D integer array)."""
    q = np.atleast_1d(np.asarray(q, dtype=np.int64))
    out = None
    for k, c in enumerate(cores):
        bit = (q >> k) & 1
        sl = c[:, bit, :]                      # (r0, nq, r1)
        sl = np.transpose(sl, (1, 0, 2))       # (nq, r0, r1)
        out = sl if out is None else np.einsum("nab,nbc->nac", out, sl)
    return out[:, 0, 0]
