import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2301_13339_b200 import qtt as Q
def mk(n, rank, decades, seed=0, pairs=False):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, n)) + 1j*rng.standard_normal((n, n))
    Qm, _ = np.linalg.qr(X)
    lam = np.zeros(n); lam[:rank] = np.logspace(0, -decades, rank)
    if pairs: lam = np.repeat(np.logspace(0, -decades, n//2), 2)
    A = (Qm * lam) @ Qm.conj().T
    return (0.5*(A + A.conj().T)).astype(np.complex128)
for mode in (0, 1):
  for n, rank, dec, pairs in [(16, 16, 3, False), (16, 8, 3, False), (20, 8, 6, False), (20, 20, 1, False), (16, 16, 3, True)]:
    A = mk(n, rank, dec, pairs=pairs)
    a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()
    lam = torch.empty(n, dtype=torch.float64, device='cuda'); U = torch.empty(2*n*n, dtype=torch.float64, device='cuda')
    sw = torch.zeros(16, dtype=torch.int32, device='cuda')
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3): Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(), s, mode=mode)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(), s, reps=50, mode=mode)
    e1.record(); torch.cuda.synchronize()
    v = sw.cpu().numpy()
    print(f"mode={mode} n={n} rank={rank} decades={dec} pairs={pairs}: {e0.elapsed_time(e1)/50*1000:.1f} us/eig, sweeps={v[0]} fallbacks={v[1]} trid cycles={list(v[2:7])} tridiag sub-phases(norm, reflector, matvec, dot+w, update)={list(v[7:12])}")
