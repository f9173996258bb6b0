import sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2301_13339_b200 import qtt as Q

n = 1 << 9                                  # 512 x 512 image, interleaved QTT bits
shp = Q.shape(2, [9, 9], "interleaved")
dec = Q.trunc(1e-3, 10)                     # TT-SVD: eps, R_max (modification 1)
fft = Q.trunc(1e-3, 8)                      # QTT-FFT / rounding: eps, Rhat_max
nb = Q.qtt_workspace_bytes(shp, dec, fft)
ws = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
f = torch.randn(n * n, dtype=torch.float64, device="cuda")
g = torch.randn(n * n, dtype=torch.float64, device="cuda")
y = torch.empty_like(f)
rep = Q.qtt_conv_full(f.data_ptr(), g.data_ptr(), y.data_ptr(), shp, dec, fft,
                      (n // 2, n // 2), (2.0 / n) ** 2, ws.data_ptr(), nb,
                      torch.cuda.current_stream().cuda_stream, report=True)
# y_j = scale * sum_i f_i g_{(j - i + shift) mod n} per axis (periodic); rep: ranks, status

print('README example ok', rep['ranks_out'][:5], rep['status_bits'])
