"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and
bench.py.

This module holds none of the method's arithmetic (no TT-SVD, FFT, Hadamard
or expansion): it only samples signals and kernels on grids.  It imports
nothing from the CUDA binding or from oracle/.

Recipes:
  * BASELINE.json configs C1-C5 — grid n = 2^b per axis, dx = 2/n,
    x_j = -1 + j dx (reading Q9); sinc(u) = sin(u)/u (reading Q14);
    signal = sinc pulses / point scatterers convolved with the same sinc
    (Q16); kernel = prod_axes sinc(w x) normalised so dx^D sum g = 1 (Q13);
    noise N(0, sigma^2) with sigma a standard deviation (Q15, F7);
    numpy Generator(PCG64(seed)), draw order positions, amplitudes, noise
    (Q17).  Periodic convolution with shift n/2 per axis, scale dx^D.
  * The paper's Examples 1-3 — midpoint
    grid x_j = -L + dx/2 + j dx, N = 2^{K-1} - 1 samples, zero padded to 2^K
    (P:339-344), kernel eq. sinc_kern1/2 normalised discretely.
"""

import numpy as np


def sinc(u):
    """sinc(u) = sin(u)/u, sinc(0) = 1 (P:185 convention, reading Q14)."""
    u = np.asarray(u, dtype=np.float64)
    out = np.ones_like(u)
    nz = u != 0.0
    out[nz] = np.sin(u[nz]) / u[nz]
    return out


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------

CONFIGS = {
    # name: (D, bits per axis, scatterers, w, eps list, seed, caps (R, Rhat))
    "c1": dict(D=1, b=12, S=3, w=40.0, eps=[1e-3], seed=1, noise="abs", sigma=0.1),
    "c2": dict(D=2, b=9, S=16, w=60.0, eps=[1e-3], seed=2, noise="rel", sigma=0.2),
    "c3": dict(D=2, b=12, S=256, w=200.0, eps=[1e-2, 1e-4], seed=3, noise="rel", sigma=0.2),
    "c4": dict(D=2, b=14, S=1024, w=800.0, eps=[1e-3], seed=4, noise="rel", sigma=0.2),
    "c5": dict(D=2, b=11, S=64, w=100.0, eps=[1e-1, 1e-2, 1e-3], seed=500, noise="rel",
               sigma=0.2, batch=64),
}

R_MAX = 10          # decomposition cap (reading Q4)
R_HAT = 8           # QTT-FFT / rounding cap (reading Q4)
CLUSTER_TOL = 1e-10  # reading Q6


def grid(b):
    n = 1 << b
    dx = 2.0 / n
    return -1.0 + dx * np.arange(n), dx


def kernel(D, b, w):
    """prod_axes sinc(w x), normalised so dx^D sum g = 1 (reading Q13)."""
    x, dx = grid(b)
    g1 = sinc(w * x)
    if D == 1:
        g = g1.copy()
    else:
        g = np.outer(g1, g1)            # g[iy, ix]
    g /= (dx ** D) * g.sum()
    return g


def signal(name, index=0, noisy=True):
    """Clean (noisy=False) or noisy signal of config `name`; `index` selects
    the image of a batch (seed = base + index).  Returns float64, 1D (n,)
    or 2D (n, n) row-major with x fastest."""
    c = CONFIGS[name]
    D, b, S, w = c["D"], c["b"], c["S"], c["w"]
    rng = np.random.Generator(np.random.PCG64(c["seed"] + index))
    x, dx = grid(b)
    n = 1 << b
    if D == 1:
        pos = rng.uniform(-0.8, 0.8, S)
        clean = sinc(w * (x[:, None] - pos[None, :])).sum(axis=1)
        sigma = c["sigma"]
        if not noisy:
            return clean
        return clean + sigma * rng.standard_normal(n)
    xs = rng.uniform(-0.8, 0.8, S)
    ys = rng.uniform(-0.8, 0.8, S)
    amp = rng.uniform(0.5, 1.0, S)
    U = sinc(w * (x[:, None] - ys[None, :]))        # rows y
    V = sinc(w * (x[:, None] - xs[None, :]))        # rows x
    clean = (U * amp[None, :]) @ V.T                 # clean[iy, ix]
    if not noisy:
        return clean
    sigma = c["sigma"] * float(np.max(np.abs(clean)))
    return clean + sigma * rng.standard_normal((n, n))


def _scatterers(name, index):
    """Draws of a 2D config in the order of signal(): positions, amplitudes;
    returns (rng positioned before the noise draw, xs, ys, amp)."""
    c = CONFIGS[name]
    rng = np.random.Generator(np.random.PCG64(c["seed"] + index))
    S = c["S"]
    xs = rng.uniform(-0.8, 0.8, S)
    ys = rng.uniform(-0.8, 0.8, S)
    amp = rng.uniform(0.5, 1.0, S)
    return rng, xs, ys, amp


def clean_block(name, index, x0, nx, y0, ny):
    """Rows y0..y0+ny-1, columns x0..x0+nx-1 of the clean 2D image of
    signal(name, index, noisy=False) (same arithmetic, restricted)."""
    c = CONFIGS[name]
    _, xs, ys, amp = _scatterers(name, index)
    x, _ = grid(c["b"])
    U = sinc(c["w"] * (x[y0:y0 + ny, None] - ys[None, :]))
    V = sinc(c["w"] * (x[x0:x0 + nx, None] - xs[None, :]))
    return (U * amp[None, :]) @ V.T


def noisy_block(name, index, x0, nx, y0, ny, clean_max, row_chunk=256):
    """The same block of signal(name, index): clean_block plus the noise
    of the full image's row-major standard_normal stream (drawn in row
    chunks up to the block's last row; sigma = sigma_rel * clean_max, with
    clean_max the maximum of |clean| over the WHOLE image)."""
    c = CONFIGS[name]
    n = 1 << c["b"]
    rng, _, _, _ = _scatterers(name, index)
    out = clean_block(name, index, x0, nx, y0, ny)
    sigma = c["sigma"] * float(clean_max)
    r = 0
    while r < y0 + ny:
        m = min(row_chunk, y0 + ny - r)
        z = rng.standard_normal((m, n))
        lo, hi = max(r, y0), min(r + m, y0 + ny)
        if lo < hi:
            out[lo - y0:hi - y0] += sigma * z[lo - r:hi - r, x0:x0 + nx]
        r += m
    return out


def kernel_block(D, b, w, x0, nx, y0=0, ny=1):
    """Block of kernel(D, b, w) (rows y0.., columns x0..; 1D: x0..x0+nx)."""
    x, dx = grid(b)
    g1 = sinc(w * x)
    tot = g1.sum() if D == 1 else g1.sum() ** 2
    if D == 1:
        return g1[x0:x0 + nx] / (dx * tot)
    return np.outer(g1[y0:y0 + ny], g1[x0:x0 + nx]) / (dx * dx * tot)


def problem(name):
    """Shape / truncation parameters of a config (caps from Q4)."""
    c = CONFIGS[name]
    b = c["b"]
    n = 1 << b
    D = c["D"]
    return dict(D=D, b=b, n=n, d=D * b, layout="1d" if D == 1 else "interleaved",
                shift=(n // 2,) * D, scale=(2.0 / n) ** D, eps=c["eps"],
                rmax=R_MAX, rhat=R_HAT, cluster_tol=CLUSTER_TOL,
                batch=c.get("batch", 1))


# ---------------------------------------------------------------------------
# Generic small random inputs for parity tests
# ---------------------------------------------------------------------------

def random_signal(shape, seed, kind="noise"):
    """kind: 'noise' (iid N(0,1)), 'smooth' (a few random sinusoids plus
    small noise) or 'lowrank' (sum of 3 separable exponentials)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = tuple(shape)
    if kind == "noise":
        return rng.standard_normal(shape)
    grids = [np.linspace(-1, 1, s, endpoint=False) for s in shape[::-1]]
    if kind == "smooth":
        out = np.zeros(shape)
        for _ in range(4):
            term = np.ones(shape)
            for ax, g in enumerate(grids):
                f = np.cos(rng.uniform(1, 12) * g + rng.uniform(0, 6.28))
                sh = [1] * len(shape)
                sh[len(shape) - 1 - ax] = shape[len(shape) - 1 - ax]
                term = term * f.reshape(sh)
            out += rng.uniform(0.5, 1.5) * term
        return out + 1e-3 * rng.standard_normal(shape)
    if kind == "lowrank":
        out = np.zeros(shape)
        for _ in range(3):
            term = np.ones(shape)
            for ax, g in enumerate(grids):
                f = np.exp(rng.uniform(-1, 1) * g)
                sh = [1] * len(shape)
                sh[len(shape) - 1 - ax] = shape[len(shape) - 1 - ax]
                term = term * f.reshape(sh)
            out += term
        return out
    raise ValueError(kind)


# ---------------------------------------------------------------------------
# The paper's worked examples (paper mode: midpoint grid, padding)
# ---------------------------------------------------------------------------

def paper_example(num, K, noisy=False, seed=0):
    """Example 1, 2 or 3 on the padded
    2^K grid.  Returns dict(f, g, N, dx, shift, scale) with f the (noisy)
    signal and g the normalised kernel, both zero padded to 2^K per axis
    (data at indices 0..N-1)."""
    N = 2 ** (K - 1) - 1
    n = 2 ** K
    rng = np.random.Generator(np.random.PCG64(seed))
    if num == 1:
        L, dx = 10.0, 20.0 / N
        x = -L + dx / 2 + dx * np.arange(N)
        f = np.exp(-(3 * x / 10) ** 2) * (0.4 * np.sin(8 * np.pi * x) - 0.7 * np.cos(6 * np.pi * x))
        res, sigma, D = 4 * dx, 0.02, 1
    elif num == 2:
        L, dx = 1.0, 2.0 / N
        x = -L + dx / 2 + dx * np.arange(N)
        f = np.exp(-(3 * x) ** 2) * (0.9 * np.sin(2 * x * np.pi / (5 * dx)) +
                                     1.4 * np.cos(x * np.pi / (3 * dx)))
        res, sigma, D = 2 * dx, 0.01, 1
    elif num == 3:
        L, dx = 1.0, 2.0 / N
        x = -L + dx / 2 + dx * np.arange(N)
        X, Y = np.meshgrid(x, x)                # X[k, j] = x_j, Y[k, j] = y_k
        f = np.exp(-((2 * X) ** 2 + (2 * Y) ** 2)) * (
            np.sin(2 * np.pi * X) - np.cos(7 * np.pi * Y) +
            np.cos(4 * np.pi * X * Y) - np.sin(3 * np.pi * X * Y))
        res, sigma, D = 2 * dx, 0.1, 2
    else:
        raise ValueError(num)
    if noisy:
        f = f + sigma * rng.standard_normal(f.shape)
    g1 = sinc(np.pi * x / res)
    g = g1 if D == 1 else np.outer(g1, g1)
    g = g / ((dx ** D) * g.sum())
    fp = np.zeros((n,) * D)
    gp = np.zeros((n,) * D)
    fp[(slice(0, N),) * D] = f
    gp[(slice(0, N),) * D] = g
    return dict(f=fp, g=gp, N=N, dx=dx, D=D, shift=((N - 1) // 2,) * D,
                scale=dx ** D, sigma=sigma)
