"""Oracle: QTT-FFT / QTT-iFFT with truncation (capped per P:370-382),
centering phase, core-wise Hadamard product (Alg. 2 Step 3) and
TT-rounding.

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

The paper delegates the QTT-FFT internals to [DKS12]; this
follows the construction fixed by SURVEY.md §8(c) O2 (radix-2 decimation in
frequency on the cores, a ROUND_LOCAL truncation after every stage, core
reversal at the end), the rounding O5 and the inverse O6.  Readings Q18-Q23,
Q28 in DESIGN.md §3.
"""

import numpy as np

from .qtt import choose_rank


def _twiddle(frac):
    """exp(-2 pi i frac) for an exact dyadic fraction (reading Q25)."""
    return np.exp(-2j * np.pi * frac)


def round_local(C, p, eps, rmax, cluster_tol, delta=None):
    """ROUND_LOCAL(p) (readings Q19/Q21/Q28).

    (i)  q = d..p+1: LQ of the r_{q-1} x 2 r_q unfolding of core q;
         core_q <- Q, core_{q-1} <- core_{q-1} L.
    (ii) tau^2 = eps^2 ||core_p||_F^2 / (d-1).
    (iii) c = p..d-1: SVD of the 2 r_{c-1} x r_c unfolding of core c,
         r = RANK(sigma^2, tau^2, R, delta_c), core_c <- U_r,
         core_{c+1} <- (Sigma_r V_r^H) core_{c+1}.
    C is a list of complex cores (r_{k-1}, 2, r_k), modified in place;
    p is 1-based.  `delta`: drop-off rule (3) instead of RANK (P:372-375:
    the same delta as the TT-SVD).
    """
    d = len(C)
    for q in range(d, p, -1):
        c = C[q - 1]
        r0, _, r1 = c.shape
        A = np.reshape(c, (r0, 2 * r1), order="F")
        Qh, R = np.linalg.qr(A.conj().T)          # A^H = Qh R
        L = R.conj().T                            # r0 x k
        Q = Qh.conj().T                           # k x 2 r1
        k = Q.shape[0]
        C[q - 1] = np.reshape(Q, (k, 2, r1), order="F")
        C[q - 2] = np.einsum("abc,cd->abd", C[q - 2], L)
    nrm2 = float(np.vdot(C[p - 1], C[p - 1]).real)
    tau2 = eps * eps * nrm2 / (d - 1)
    for c in range(p, d):
        core = C[c - 1]
        r0, _, r1 = core.shape
        A = np.reshape(core, (2 * r0, r1), order="F")
        U, s, Vh = np.linalg.svd(A, full_matrices=False)
        r = choose_rank(s * s, tau2, rmax, cluster_tol, delta)
        C[c - 1] = np.reshape(U[:, :r], (r0, 2, r), order="F")
        SV = s[:r, None] * Vh[:r, :]
        C[c] = np.einsum("ab,bcd->acd", SV, C[c])
    return C


def qfft(cores, axes, bits, eps, rmax, cluster_tol=1e-10, delta=None, stages=None):
    """Unnormalised per-axis DFT (omega = e^{-2 pi i / 2^{b_a}})
    of a QTT tensor, truncated after every stage.

    axes: the (axis, bit) descriptor of every position (oracle.qtt.
    axes_descriptor); bits: bits per axis.  For p = d..1 with a = axis(p),
    t = bit(p), stage s = b_a - t + 1:
      p = d:  core_d[:, al, :] <- core_d[:,0,:] + (-1)^al core_d[:,1,:]
      p < d:  core_p[:, al, :] <- [core_p[:,0,:] | (-1)^al core_p[:,1,:]];
              core_q <- blockdiag(core_q, phi_q core_q), p < q < d;
              core_d <- vstack(core_d, phi_d core_d);
              phi_q(be) = exp(-2 pi i be 2^{m-1} / 2^s), m = b_a + 1 - bit(q),
              for axis(q) = a, else 1;  then ROUND_LOCAL(p).
    Finally the cores are reversed (core'_q = core_{d+1-q}, rank indices
    swapped), which puts frequency bit m of axis a at the slot of bit m of
    the *other* group in 2D (F8) — F and G share that layout.

    `stages` (test hook): stop after that many stages, before the reversal.
    """
    C = [np.array(c, dtype=np.complex128) for c in cores]
    d = len(C)
    done = 0
    for p in range(d, 0, -1):
        if stages is not None and done == stages:
            return C
        a, t = axes[p - 1]
        s = bits[a] - t + 1
        if p == d:
            c = C[d - 1]
            C[d - 1] = np.stack([c[:, 0, :] + c[:, 1, :],
                                 c[:, 0, :] - c[:, 1, :]], axis=1)
            done += 1
            continue
        c = C[p - 1]
        r0, _, r1 = c.shape
        n = np.zeros((r0, 2, 2 * r1), dtype=np.complex128)
        n[:, 0, :r1] = c[:, 0, :]
        n[:, 0, r1:] = c[:, 1, :]
        n[:, 1, :r1] = c[:, 0, :]
        n[:, 1, r1:] = -c[:, 1, :]
        C[p - 1] = n

        def phi(q, be):
            aq, tq = axes[q - 1]
            if aq != a or be == 0:
                return 1.0 + 0.0j
            m = bits[a] + 1 - tq
            return _twiddle(2.0 ** (m - 1 - s))

        for q in range(p + 1, d):
            c = C[q - 1]
            r0, _, r1 = c.shape
            n = np.zeros((2 * r0, 2, 2 * r1), dtype=np.complex128)
            for be in (0, 1):
                n[:r0, be, :r1] = c[:, be, :]
                n[r0:, be, r1:] = phi(q, be) * c[:, be, :]
            C[q - 1] = n
        c = C[d - 1]
        r0 = c.shape[0]
        n = np.zeros((2 * r0, 2, 1), dtype=np.complex128)
        for be in (0, 1):
            n[:r0, be, :] = c[:, be, :]
            n[r0:, be, :] = phi(d, be) * c[:, be, :]
        C[d - 1] = n
        round_local(C, p, eps, rmax, cluster_tol, delta)
        done += 1
    if stages is not None:
        return C
    return [np.ascontiguousarray(C[d - 1 - q].transpose(2, 1, 0)) for q in range(d)]


def center(C, axes, bits, shift):
    """Shift the (transformed) kernel by c_a per axis: multiply slice 1 of the
    core holding frequency bit m of axis a by exp(+2 pi i c_a 2^{m-1}/2^{b_a})
    (DFT shift theorem applied to eq. dconv's index offset, P:95 / P:157;
    reading Q10).  After qfft's reversal, slot q holds
    frequency bit m = b_a + 1 - bit(d+1-q) of axis a = axis(d+1-q).
    """
    d = len(C)
    out = [c.copy() for c in C]
    for q in range(1, d + 1):
        a, t = axes[d - q]
        m = bits[a] + 1 - t
        b = bits[a]
        num = (int(shift[a]) << (m - 1)) % (1 << b)     # exact dyadic phase
        if num == 0:
            continue
        out[q - 1][:, 1, :] *= np.exp(2j * np.pi * num / float(1 << b))
    return out


def hadamard(F, G):
    """Core-wise Kronecker product: Z_k[(a,a'), al, (b,b')] =
    F_k[a, al, b] G_k[a', al, b'] (Hadamard product in TT);
    ranks multiply.  Combined index a' + r_G a (C order)."""
    Z = []
    for f, g in zip(F, G):
        z = np.einsum("iaj,kal->ikajl", f, g)
        Z.append(z.reshape(f.shape[0] * g.shape[0], 2, f.shape[2] * g.shape[2]))
    return Z


def round_full(Z, eps, rmax, cluster_tol=1e-10, delta=None):
    """TT-rounding ROUND_FULL = ROUND_LOCAL(1) (reading Q20/Q21, O5)."""
    C = [np.array(c, dtype=np.complex128) for c in Z]
    return round_local(C, 1, eps, rmax, cluster_tol, delta)


def qifft(C, axes, bits, eps, rmax, cluster_tol=1e-10, delta=None):
    """QTT-iFFT (IDFT P:118-125): conj, qfft, conj, scale core_1
    by 2^{-d} = 1/N^D (reading Q23, O6)."""
    d = len(C)
    out = qfft([np.conj(c) for c in C], axes, bits, eps, rmax, cluster_tol, delta)
    out = [np.conj(c) for c in out]
    out[0] = out[0] * (2.0 ** (-d))
    return out
