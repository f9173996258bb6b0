import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2301_13339_b200 import qtt as Q
def mk(n, rank, decades, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, n)) + 1j*rng.standard_normal((n, n))
    Qm, _ = np.linalg.qr(X)
    lam = np.zeros(n); lam[:rank] = np.logspace(0, -decades, rank)
    A = (Qm * lam) @ Qm.conj().T
    return (0.5*(A + A.conj().T)).astype(np.complex128)
for n, rank, dec in [(16, 16, 3), (16, 8, 3), (20, 8, 6), (20, 20, 1)]:
    A = mk(n, rank, dec)
    a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()
    lam = torch.empty(n, dtype=torch.float64, device='cuda'); U = torch.empty(2*n*n, dtype=torch.float64, device='cuda')
    sw = torch.zeros(8, dtype=torch.int32, device='cuda')
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3): Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(), s)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(), s, reps=50)
    e1.record(); torch.cuda.synchronize()
    v = sw.cpu().numpy()
    print(f"n={n} rank={rank} decades={dec}: {e0.elapsed_time(e1)/50*1000:.1f} us/eig, sweeps64={v[0]} sweeps32={v[1]} cycles fp32={v[2]} basis={v[3]} fp64={v[4]} sort={v[5]}")
