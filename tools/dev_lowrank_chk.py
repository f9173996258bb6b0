import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2301_13339_b200 import qtt as Q
Q.LIB_PATH = '/root/repo/build/libqtt_chk.so'
import oracle as O
from gpu_util import *
d = 14; n = 1 << d
x = np.arange(n) / n
f = np.cos(17 * 2 * np.pi * x) + 0.3 * np.sin(3 * 2 * np.pi * x + 0.2) + 0.2
g = np.cos(3 * 2 * np.pi * x) + 0.5 * np.cos(17 * 2 * np.pi * x + 1.0)
eps = 1e-6
y, rep = gpu_conv_full(f, g, "1d", (eps, 10, 1e-10), (eps, 8, 1e-10), (n // 2,), 1.0 / n)
print("status bits", rep["status_bits"], rep["ranks_out"])
