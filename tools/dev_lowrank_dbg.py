import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O
from gpu_util import *
d = 14; n = 1 << d
x = np.arange(n) / n
f = np.cos(17 * 2 * np.pi * x) + 0.3 * np.sin(3 * 2 * np.pi * x + 0.2) + 0.2
g = np.cos(3 * 2 * np.pi * x) + 0.5 * np.cos(17 * 2 * np.pi * x + 1.0)
eps = 1e-6
for name, v in (("f", f), ("g", g)):
    ref = O.tt_svd(v, eps, 10, 1e-10)
    tt = gpu_decompose(v, "1d", eps, 10)
    full = gpu_full(tt, v)
    print(name, "ranks gpu", tt.ranks(), "oracle", O.ranks_of(ref), "rel", np.linalg.norm(full - O.full(ref)) / np.linalg.norm(v))
    # forward transform of oracle cores on the GPU vs oracle
    axes = O.axes_descriptor(1, [d], "1d")
    Fh = O.qfft(ref, axes, [d], eps, 8, 1e-10)
    tth = gpu_tt_from_cores(ref, v, "1d")
    th = gpu_transform(tth, None, eps, 8)
    got = gpu_full(th, v, imag=True)
    want = O.full(Fh)
    print(name, "qfft ranks gpu", th.ranks(), "oracle", O.ranks_of(Fh), "rel", np.linalg.norm(got - want) / np.linalg.norm(want))
c, h = n // 2, 1.0 / n
y, rep = gpu_conv_full(f, g, "1d", (eps, 10, 1e-10), (eps, 8, 1e-10), (c,), h)
ref, info = O.conv_pipeline(f, g, "1d", (eps, 10, 1e-10), (eps, 8, 1e-10), (c,), h, return_info=True)
print("conv rel", np.linalg.norm(y - ref) / np.linalg.norm(ref), "status", rep["status_bits"])
print("ranks out gpu", rep["ranks_out"], "oracle", O.ranks_of(info["Y"]))
print({k: (O.ranks_of(v) if isinstance(v, list) else None) for k, v in info.items()})
# round(hadamard) from oracle F^, G^ on GPU
Fh, Gh = info["Fh"], info["Gh"]
tf = gpu_tt_from_cores(Fh, f, "1d"); tg = gpu_tt_from_cores(Gh, g, "1d")
w = ws(256 << 20)
ty = Q.qtt_convolve(tf, tg, Q.trunc(eps, 8), None, h, w.data_ptr(), 256 << 20, stream(), ws_owner=w)
print("convolve-from-oracle-spectra ranks", ty.ranks())
Z = info["Z"]
tz = gpu_tt_from_cores(Z, f, "1d")
ti = gpu_transform(tz, None, eps, 8, inverse=True, scale=h)
got = gpu_full(ti, f, imag=True)
want = h * O.full(info["Y"]) if False else None
print("inverse-from-oracle-Z ranks", ti.ranks(), "oracle Y", O.ranks_of(info["Y"]))
