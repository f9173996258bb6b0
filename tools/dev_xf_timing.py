# per-phase cycles of the transform kernel (needs libqtt built with -DQTT_XF_TIMING)
import sys, ctypes, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2301_13339_b200 import synth, qtt as Q
import os; Q.LIB_PATH = os.environ.get('QTT_LIB', '/root/repo/build_tmp/libqtt_xf.so')
from gpu_util import *
def run(x, label, inverse=False):
    tt = gpu_decompose(x, "interleaved", 1e-3, 10)
    fft = Q.trunc(1e-3, 8)
    nb = 64 << 20
    w = ws(nb)
    st = torch.zeros(1, dtype=torch.int32)
    th = Q.qtt_transform(tt, fft, 0, None, 1.0, w.data_ptr(), nb, stream(), ws_owner=w)
    torch.cuda.synchronize()
    raw = w.cpu().numpy().view(np.int64)
    d = int(np.log2(x.size))
    off = 0
    def take(nbytes):
        nonlocal off
        off = (off + 255) & ~255; o = off; off += nbytes; return o
    take(d*512*16); take(64*4)
    gr = take(30*400*16)
    base = (gr + (30*400 - 8)*16)//8
    cyc = raw[base:base+6]
    names = ['GR chain','K formation','eig values','rank/vectors/push','tail','load GR']
    tot = cyc.sum()
    print(label, 'total %.1f us' % (tot/1.965e3), ' '.join(f"{n_}={c/1.965e3:.0f}us" for n_, c in zip(names, cyc)))
    # status bits (fallbacks) live in the decompose workspace status word
    return th
run(synth.signal("c2"), "F(c2)")
run(synth.kernel(2, 9, 60.0), "G(c2 kernel)")
