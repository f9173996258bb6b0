# feed the Gram matrices of ROUND_FULL(Z) (low-rank convolution case) to the GPU eigensolver
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O
from paper_2301_13339_b200 import qtt as Q
d = 14; n = 1 << d
x = np.arange(n) / n
f = np.cos(17 * 2 * np.pi * x) + 0.3 * np.sin(3 * 2 * np.pi * x + 0.2) + 0.2
g = np.cos(3 * 2 * np.pi * x) + 0.5 * np.cos(17 * 2 * np.pi * x + 1.0)
eps = 1e-6
_, info = O.conv_pipeline(f, g, "1d", (eps, 10, 1e-10), (eps, 8, 1e-10), (n // 2,), 1.0 / n, return_info=True)
Z = O.hadamard(info["Fh"], info["Gh"])
C = [c.copy() for c in Z]
# right orthogonalisation (LQ) d..2
for q in range(d - 1, 0, -1):
    r0, _, r1 = C[q].shape
    M = C[q].reshape(r0, 2 * r1, order="F")
    Qm, R = np.linalg.qr(M.conj().T)
    C[q] = Qm.conj().T.reshape(-1, 2, r1, order="F")
    C[q - 1] = np.einsum("aib,bc->aic", C[q - 1], R.conj().T)
tr = None
def gpu(K, mode):
    m = K.shape[0]
    a = torch.from_numpy(np.ascontiguousarray(K.T).view(np.float64).copy()).cuda()
    lam = torch.empty(m, dtype=torch.float64, device='cuda'); U = torch.empty(2*m*m, dtype=torch.float64, device='cuda')
    sw = torch.zeros(16, dtype=torch.int32, device='cuda')
    Q.qtt_debug_eigh(a.data_ptr(), m, lam.data_ptr(), U.data_ptr(), sw.data_ptr(), torch.cuda.current_stream().cuda_stream, mode=mode)
    torch.cuda.synchronize()
    return lam.cpu().numpy(), U.cpu().numpy().view(np.complex128).reshape(m, m).T, int(sw[1])
for c in range(d - 1):
    r0, _, r1 = C[c].shape
    M = C[c].reshape(2 * r0, r1, order="F")
    K = M @ M.conj().T
    if tr is None:
        tr = np.trace(K).real
    lam, U = np.linalg.eigh(K); lam, U = lam[::-1], U[:, ::-1]
    r = O.rank_rule(lam[:min(2 * r0, r1)], eps * eps * tr / (d - 1), 8, 1e-10)
    lg, ug, fb = gpu(K, r + 1)
    nrm = np.linalg.norm(K)
    res = np.linalg.norm(K @ ug[:, :r] - ug[:, :r] * lg[:r]) / nrm
    orth = np.linalg.norm(ug[:, :r].conj().T @ ug[:, :r] - np.eye(r))
    print(f"cut {c+1}: n={2*r0} r={r} lam err {np.abs(lg-lam).max()/nrm:.1e} res {res:.1e} orth {orth:.1e} fb {fb}  lam={np.array2string(lam[:6]/lam[0], precision=3)}")
    Ur = U[:, :r]
    C[c] = Ur.reshape(r0, 2, r, order="F")
    S = Ur.conj().T @ M
    C[c + 1] = np.einsum("ab,bic->aic", S, C[c + 1])
