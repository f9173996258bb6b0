"""The small Hermitian eigensolver behind every truncated SVD of the GPU path
(tridiagonal + multisection + twisted vectors, Jacobi fallback) against
numpy.linalg.eigh (LAPACK) on the spectra the cut Grams K = M GR M^H have:
graded, rank-deficient (null clusters) and exactly degenerate pairs.
Eigenvalues to ~1e-15 ||K||, eigenvectors of separated eigenvalues to
eps ||K|| / gap, invariant subspaces of clusters exactly spanned."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2301_13339_b200 import qtt as Q  # noqa: E402


def _gpu_eigh(A, mode):
    n = A.shape[0]
    a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()  # column-major
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    U = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
    sw = torch.zeros(16, dtype=torch.int32, device="cuda")
    Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(),
                     torch.cuda.current_stream().cuda_stream, mode=mode)
    torch.cuda.synchronize()
    u = U.cpu().numpy().view(np.complex128).reshape(n, n).T
    return lam.cpu().numpy(), u, sw.cpu().numpy()


def _matrix(n, lam, cplx, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
    Qm, _ = np.linalg.qr(X)
    A = (Qm * lam) @ Qm.conj().T
    return (0.5 * (A + A.conj().T)).astype(np.complex128)


CASES = [
    ("graded16", 16, lambda n: np.logspace(0, -2, n), True),
    ("graded20", 20, lambda n: np.logspace(0, -10, n), True),
    ("graded32_real", 32, lambda n: np.logspace(0, -12, n), False),
    ("odd7", 7, lambda n: np.logspace(0, -14, n), True),
    ("one", 1, lambda n: np.ones(n), True),
    ("rank8_of16", 16, lambda n: np.r_[np.logspace(0, -3, 8), np.zeros(8)], True),
    ("rank2_of16", 16, lambda n: np.r_[1.0, 0.3, np.zeros(14)], True),
    ("degenerate_pairs", 16, lambda n: np.repeat(np.logspace(0, -4, 8), 2), True),
    ("triple_cluster", 12, lambda n: np.r_[1.0, 0.5, 0.5, 0.5, np.logspace(-1, -6, 8)], True),
]


@pytest.mark.parametrize("mode", [0, 1], ids=["tridiagonal", "jacobi"])
@pytest.mark.parametrize("name,n,spec,cplx", CASES, ids=[c[0] for c in CASES])
def test_small_eigensolver_matches_lapack(mode, name, n, spec, cplx):
    lam_true = np.sort(spec(n))[::-1]
    A = _matrix(n, lam_true, cplx, n + 7)
    lg, ug, sw = _gpu_eigh(A, mode)
    lw, uw = np.linalg.eigh(A)
    lw, uw = lw[::-1], uw[:, ::-1]
    nrm = np.linalg.norm(A)
    assert np.max(np.abs(lg - lw)) <= 2e-15 * n * nrm
    # orthonormality: 1e-12 inside a group of (numerically) equal eigenvalues;
    # across groups the Davis-Kahan bound the subspace check below uses,
    # 50 eps n ||A|| / |lambda_i - lambda_j| (a null vector of a rank-deficient
    # Gram against a kept vector 1e-3 ||A|| away may overlap ~1e-12)
    O = np.abs(ug.conj().T @ ug - np.eye(n))
    sep = np.abs(lw[:, None] - lw[None, :])
    bound = np.where(sep <= 1e-9 * nrm, 1e-12, np.maximum(1e-12, 50 * 1.1e-16 * n * nrm / np.maximum(sep, 1e-300)))
    assert np.all(O <= bound), float((O / bound).max())
    assert np.linalg.norm(A @ ug - ug * lg) <= 1e-14 * n * nrm
    # invariant subspaces of groups of (numerically) equal eigenvalues agree
    k = 0
    while k < n:
        j = k + 1
        while j < n and abs(lw[j] - lw[j - 1]) <= 1e-9 * nrm:
            j += 1
        gap = min([abs(lw[k] - lw[k - 1])] if k > 0 else [np.inf])
        gap = min(gap, abs(lw[j - 1] - lw[j]) if j < n else np.inf)
        if gap > 1e-12 * nrm:
            P = uw[:, k:j] @ uw[:, k:j].conj().T
            Pg = ug[:, k:j] @ ug[:, k:j].conj().T
            assert np.linalg.norm(P - Pg) <= max(1e-12, 50 * 1.1e-16 * n * nrm / gap)
        k = j
    if mode == 1:
        assert sw[0] <= 20


@pytest.mark.parametrize("n", [4, 12, 16])
@pytest.mark.parametrize("mode", [0, 3], ids=["all_vectors", "top2_vectors"])
def test_nearly_diagonal_gram_with_rounding_asymmetry(n, mode):
    """The cut Grams K = M GR M^H are Hermitian only to rounding.  For a
    nearly diagonal K (near-degenerate pairs, off-diagonal ~1e-18 ||K||) the
    rounding asymmetry is as large as the reflector columns themselves; the
    solver must still return the eigenpairs of K (regression: a reflector
    formula that assumed exact symmetry lost ~10% of K here)."""
    rng = np.random.default_rng(n)
    d = np.repeat([1.1259e15, 4.0532e14], n // 2)[:n] * (1 + 1e-14 * rng.standard_normal(n))
    E = 1e-3 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))  # not Hermitian
    A = np.diag(d).astype(np.complex128) + E
    lg, ug, _ = _gpu_eigh(A, mode)
    H = 0.5 * (A + A.conj().T)
    lw = np.linalg.eigvalsh(H)[::-1]
    nrm = np.linalg.norm(A)
    assert np.max(np.abs(lg - lw)) <= 1e-14 * nrm
    k = n if mode == 0 else 2
    # backward-stable to ~1e-13 ||K|| even where a pair is split by only ~eps ||K||
    assert np.linalg.norm(H @ ug[:, :k] - ug[:, :k] * lg[:k]) <= 1e-12 * nrm


def test_reflector_column_with_tiny_leading_entry():
    """A Gram from the rounding of a low-rank convolution (captured input;
    expected values from LAPACK): the first reflector column has |x_0| ~
    2e-3 |x| with |x|^2 ~ 4e-57 ||A||^2.  tau = 1/(sig (sig + |x_0|)) must use
    the true |x_0| or the reflector is not unitary (regression)."""
    A = np.array([
        [1531223873305724.5 + 0.030530668773954436j, -3.0459277739610207e-16 + 1.5869363548134762e-16j,
         6.3977605118900718e-16 - 7.8462981843276434e-16j, 1.3105847166115026e-13 - 3.3426406628489761e-14j],
        [-3.0459277739610202e-16 - 1.5869363548134792e-16j, 1.1180514300345477e-44 + 7.3921320910909081e-61j,
         -1.1583067596956201e-44 - 9.3951900008114141e-46j, -2.0880786016810227e-16 - 4.1180467773050174e-15j],
        [6.3977605118900709e-16 + 7.8462981843276425e-16j, -1.1583067596956201e-44 + 9.3951900008114001e-46j,
         1.2416893482199729e-44 + 7.2213845986493022e-61j, 5.9564751273308451e-16 + 4.199201165122222e-15j],
        [1.5808276109183045e-13 + 3.0227753260396385e-14j, -2.0880786016810259e-16 + 4.1180467773050182e-15j,
         5.9564751273308471e-16 - 4.1992011651222228e-15j, 1531223873305665 + 0.043046907873092941j]])
    H = 0.5 * (A + A.conj().T)
    lw = np.linalg.eigvalsh(H)[::-1]
    nrm = np.linalg.norm(A)
    for mode in (0, 3):
        lg, ug, _ = _gpu_eigh(A, mode)
        assert np.max(np.abs(lg - lw)) <= 1e-14 * nrm
        k = 4 if mode == 0 else 2
        assert np.linalg.norm(H @ ug[:, :k] - ug[:, :k] * lg[:k]) <= 1e-12 * nrm
