# stress the production eigensolver (mode 0) on degenerate Hermitian matrices
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2301_13339_b200 import qtt as Q
def run(A, mode=0):
    n = A.shape[0]
    a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()
    lam = torch.empty(n, dtype=torch.float64, device='cuda'); U = torch.empty(2*n*n, dtype=torch.float64, device='cuda')
    sw = torch.zeros(16, dtype=torch.int32, device='cuda')
    Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(), torch.cuda.current_stream().cuda_stream, mode=mode)
    torch.cuda.synchronize()
    l = lam.cpu().numpy(); u = U.cpu().numpy().view(np.complex128).reshape(n, n).T
    ref = np.sort(np.linalg.eigvalsh(A))[::-1]
    nrm = np.linalg.norm(A)
    k = min(n, 8) if mode == 0 else min(n, mode - 1)
    res = np.linalg.norm(A @ u[:, :k] - u[:, :k] * l[:k]) / max(nrm, 1e-300)
    return np.abs(l - ref).max() / max(nrm, 1e-300), res, int(sw[1])
rng = np.random.default_rng(0)
cases = []
for n in (4, 8, 16, 20):
    for r in (1, 2, 3, n // 2):
        X = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
        cases.append((f"n={n} rank={r}", X @ X.conj().T))
    # zero rows/cols in the middle
    X = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
    X[1:n//2] = 0
    cases.append((f"n={n} zero-block", X @ X.conj().T))
    D = np.diag(rng.standard_normal(n)).astype(complex)
    cases.append((f"n={n} diagonal", D))
    cases.append((f"n={n} zero", np.zeros((n, n), complex)))
for n in (8, 12, 16):
    for m in (1, 2, 3):
        # decoupled leading block of size m (zero sub-column at step m-1)
        X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        H = X @ X.conj().T
        H[:m, m:] = 0; H[m:, :m] = 0
        cases.append((f"n={n} split@{m}", H))
        # low rank with a zero leading column
        Y = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
        Y[:m] = 0
        cases.append((f"n={n} lr2 zero-lead{m}", Y @ Y.conj().T))
    # Kronecker-like rank structure: rank-4 product of two rank-2 factors
    a = rng.standard_normal((4, 2)) + 1j * rng.standard_normal((4, 2))
    b = rng.standard_normal((n // 4, 2)) + 1j * rng.standard_normal((n // 4, 2))
    K = np.kron(a @ a.conj().T, b @ b.conj().T)
    cases.append((f"n={n} kron", K))
for name, A in cases:
  for mode in (0, 2, 3, 5):
    e, r, fb = run(A, mode)
    print(f"{name:22s} mode {mode} eig err {e:.1e} residual {r:.1e} fallback {fb} {'BAD' if (e > 1e-12 or r > 1e-10) else ''}")
