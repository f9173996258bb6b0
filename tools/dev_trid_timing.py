# per-sub-phase cycles of the single-warp tridiagonalisation (lib built with -DQTT_TRID_TIMING)
import sys, os
sys.path.insert(0, '/root/repo')
from paper_2301_13339_b200 import qtt as Q
Q.LIB_PATH = os.environ.get("QTT_LIB", '/root/repo/build/libqtt_trid.so')
exec(open('/root/repo/tools/dev_eig_time.py').read().split("for mode in (0, 1):")[0])
import numpy as np, torch
for n, mode in ((16, 0), (16, 256), (20, 256), (20, 0)):
    A = mk(n, n, 3)
    a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()
    lam = torch.empty(n, dtype=torch.float64, device='cuda'); U = torch.empty(2*n*n, dtype=torch.float64, device='cuda')
    sw = torch.zeros(16, dtype=torch.int32, device='cuda')
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3): Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(), s, mode=mode)
    torch.cuda.synchronize()
    v = sw.cpu().numpy()
    print(f"n={n} nmax={'20' if mode else ('16' if n <= 16 else '32')}: phases(trid, values, twist, mgs, back)={list(v[2:7])} trid sub(y+bar, reduce+bar, scalars+publish, update+bar, values-loop)={list(v[7:12])}")
