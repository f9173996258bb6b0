import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2301_13339_b200 import qtt as Q
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(0)
X = rng.standard_normal((n, n)) + 1j*rng.standard_normal((n, n)); Qm,_ = np.linalg.qr(X)
lam = np.logspace(0, -3, n)
A = ((Qm * lam) @ Qm.conj().T).astype(np.complex128)
a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()
l = torch.empty(n, dtype=torch.float64, device='cuda'); U = torch.empty(2*n*n, dtype=torch.float64, device='cuda')
sw = torch.zeros(8, dtype=torch.int32, device='cuda')
for _ in range(2): Q.qtt_debug_eigh(a.data_ptr(), n, l.data_ptr(), U.data_ptr(), sw.data_ptr(), 0, reps=20, mode=mode)
torch.cuda.synchronize(); print('ok', sw.cpu().numpy())
