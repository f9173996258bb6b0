"""Oracle: Alg. 2 QTT convolution end to end, SURVEY §8(c) O8.

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.
"""

import numpy as np

from .qtt import axes_descriptor, to_qtt, from_qtt, tt_svd, full
from .qfft import qfft, qifft, center, hadamard, round_full


def conv_pipeline(f, g, layout, dec, fft, shift, scale, return_info=False, rsvd=None):
    """y_j = scale * sum_i f_i g_{(j - i + shift) mod n} per axis, computed as
    Alg. 2: Step 1 reshape to 2x..x2, Step 2 max-rank TT-SVD of
    both (Alg. 1 + mod (1)), Step 3 QiFFT(QFFT(F) (.) QFFT(G))
     with the centering phase on G (O3) and ROUND_FULL after the
    Hadamard product (Q20), Step 4 Full (Alg. 3), real part (Q22).

    f, g: float64 arrays, 1D (n,) or 2D (n, n) row-major with x fastest.
    layout: '1d' | 'interleaved' | 'concat'.
    dec, fft: (eps, rmax, cluster_tol) for the TT-SVD and for QFFT/round/QiFFT,
    or (eps, rmax, cluster_tol, delta) for the SV drop-off rule (3) with the
    same delta in both (eps unused, rmax = capacity cap).
    shift: per-axis integer shift (tuple, x first); scale: h = dx^D (Q12).
    """
    f = np.asarray(f, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    D = f.ndim
    shape = f.shape
    bits = [int(np.log2(s)) for s in (shape[::-1] if D == 2 else shape)]
    axes = axes_descriptor(D, bits, "1d" if D == 1 else layout)
    lay = "1d" if D == 1 else layout
    vf = to_qtt(f, lay)
    vg = to_qtt(g, lay)
    # rsvd = (p, seed_f, seed_g): max-rank TT-RSVD (modification (2)) for the
    # TT-SVD of f and g (reading N2: the QTT-FFT / rounding keep (1))
    F = tt_svd(vf, *dec, rsvd=None if rsvd is None else (rsvd[0], rsvd[1]))
    G = tt_svd(vg, *dec, rsvd=None if rsvd is None else (rsvd[0], rsvd[2]))
    Fh = qfft(F, axes, bits, *fft)
    Gh = qfft(G, axes, bits, *fft)
    Gh = center(Gh, axes, bits, shift)
    Z = round_full(hadamard(Fh, Gh), *fft)
    Y = qifft(Z, axes, bits, *fft)
    yq = scale * np.real(full(Y))
    y = from_qtt(yq, shape, lay)
    if return_info:
        return y, {"F": F, "G": G, "Fh": Fh, "Gh": Gh, "Z": Z, "Y": Y}
    return y
