"""The CTA Jacobi eigensolver (every truncated SVD of the GPU path) against
numpy.linalg.eigh (LAPACK) on graded Hermitian PSD spectra like the cut Grams
K = M GR M^H: eigenvalues to 1e-15 ||K||, eigenvectors of well-separated
eigenvalues to eps ||K|| / gap."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2301_13339_b200 import qtt as Q  # noqa: E402


def _gpu_eigh(A):
    n = A.shape[0]
    a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()  # column-major
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    U = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
    sw = torch.zeros(8, dtype=torch.int32, device="cuda")
    Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    u = U.cpu().numpy().view(np.complex128).reshape(n, n).T
    return lam.cpu().numpy(), u, int(sw[0].item())


@pytest.mark.parametrize("n,decades,cplx", [(16, 2, True), (20, 10, True), (32, 12, False),
                                            (7, 14, True), (1, 0, True)])
def test_jacobi_matches_lapack(n, decades, cplx):
    rng = np.random.default_rng(n + decades)
    X = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
    Qm, _ = np.linalg.qr(X)
    lam = np.logspace(0, -decades, n)
    A = (Qm * lam) @ Qm.conj().T
    A = (0.5 * (A + A.conj().T)).astype(np.complex128)
    lg, ug, sweeps = _gpu_eigh(A)
    lw, uw = np.linalg.eigh(A)
    lw, uw = lw[::-1], uw[:, ::-1]
    assert np.max(np.abs(lg - lw)) <= 1e-15 * n * np.abs(lw).max()
    assert np.allclose(ug.conj().T @ ug, np.eye(n), atol=1e-13)
    assert np.linalg.norm(A @ ug - ug * lg) <= 1e-14 * n * np.linalg.norm(A)
    for k in range(n):
        gap = min([abs(lw[k] - lw[j]) for j in range(n) if j != k] or [1.0])
        ang = 1 - abs(np.vdot(ug[:, k], uw[:, k]))
        assert ang <= max(1e-13, (4e-16 * n * lw[0] / gap) ** 2 * 10)
    assert sweeps <= 20
