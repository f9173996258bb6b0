# per-phase cycles of the transform kernel (needs libqtt built with -DQTT_XF_TIMING)
import sys, ctypes, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2301_13339_b200 import synth, qtt as Q
Q.LIB_PATH = '/root/repo/build/libqtt_timing.so'
from gpu_util import *
x = synth.signal("c2")
tt = gpu_decompose(x, "interleaved", 1e-3, 10)
fft = Q.trunc(1e-3, 8)
nb = 64 << 20
w = ws(nb)
th = Q.qtt_transform(tt, fft, 0, None, 1.0, w.data_ptr(), nb, stream(), ws_owner=w)
torch.cuda.synchronize()
# gr scratch of the first transform starts after the output TT carve: find it by scanning the tail marker region
raw = w.cpu().numpy().view(np.int64)
# XfProb.gr = after output TT (d*512 complex + 64 ints, 256-aligned) -> compute offsets like the carver
d = 18
off = 0
def take(nbytes):
    global off
    off = (off + 255) & ~255; o = off; off += nbytes; return o
take(d*512*16); take(64*4)
gr = take(30*400*16)
base = (gr + (30*400 - 8)*16)//8
cyc = raw[base:base+6]
names = ['GR chain','K formation','eig','rank/push/next-E','tail','load GR']
tot = cyc.sum()
for n_, c in zip(names, cyc): print(f"{n_:18s} {c/1.965e3:10.1f} us  {100*c/tot:5.1f}%")
print('total', tot/1.965e3, 'us')
