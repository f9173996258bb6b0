"""Helpers for the GPU tests: device buffers (torch is only the allocator) and
calls through the C ABI (paper_2301_13339_b200.qtt)."""

import numpy as np
import torch

from paper_2301_13339_b200 import qtt as Q


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def ws(nbytes):
    return torch.empty(int(nbytes) + 256, dtype=torch.uint8, device="cuda")


def stream():
    return torch.cuda.current_stream().cuda_stream


def layout_of(x, layout):
    return "1d" if x.ndim == 1 else layout


def shape_of(x, layout, batch=1, f_stride=0, g_stride=0, y_stride=0):
    if x.ndim == 1:
        return Q.shape(1, [int(np.log2(x.shape[0])), 0], "1d", batch, f_stride, g_stride, y_stride)
    b = int(np.log2(x.shape[-1]))
    return Q.shape(2, [b, b], layout, batch, f_stride, g_stride, y_stride)


def gpu_decompose(x, layout, eps, rmax, ctol=1e-10):
    """TT-SVD on the GPU; returns (TT handle, keepalive)."""
    xd = dev(x)
    shp = shape_of(x, layout)
    dec = Q.trunc(eps, rmax, ctol)
    fft = Q.trunc(eps, min(rmax, 8), ctol)
    nb = Q.qtt_workspace_bytes(shp, dec, fft)
    w = ws(nb)
    tt = Q.qtt_decompose(xd.data_ptr(), shp, dec, w.data_ptr(), nb, stream(), ws_owner=(w, xd))
    return tt


def gpu_decompose_policy(x, layout, dec):
    """TT-SVD on the GPU with a full truncation tuple (eps, rmax, ctol[, delta[, rsvd]])."""
    xd = dev(x)
    shp = shape_of(x, layout)
    D = Q.trunc(*dec)
    fft = Q.trunc(dec[0], min(dec[1], 8), dec[2])
    nb = Q.qtt_workspace_bytes(shp, D, fft)
    w = ws(nb)
    return Q.qtt_decompose(xd.data_ptr(), shp, D, w.data_ptr(), nb, stream(), ws_owner=(w, xd))


def gpu_full(tt, like, imag=False):
    """Expand a TT handle to a full array shaped like `like` (complex if imag)."""
    n = like.size
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    yi = torch.empty(n, dtype=torch.float64, device="cuda") if imag else None
    w = ws(1 << 22)
    Q.qtt_to_full(tt, y.data_ptr(), w.data_ptr(), 1 << 22, stream(),
                  yi.data_ptr() if imag else None)
    torch.cuda.synchronize()
    out = y.cpu().numpy().reshape(like.shape)
    if imag:
        out = out + 1j * yi.cpu().numpy().reshape(like.shape)
    return out


def gpu_transform(tt, layout_shape_x, eps, rmax, inverse=False, shift=None, scale=1.0, ctol=1e-10):
    fft = Q.trunc(eps, rmax, ctol)
    nb = 64 << 20
    w = ws(nb)
    return Q.qtt_transform(tt, fft, inverse, shift, scale, w.data_ptr(), nb, stream(), ws_owner=w)


def gpu_conv_full(f, g, layout, dec, fft, shift, scale, batch=1, shared_g=True, report=True):
    fd = dev(f)
    gd = dev(g)
    n = f.size // batch
    shp = shape_of(f.reshape((batch,) + f.shape[1:])[0] if batch > 1 else f, layout, batch,
                   f_stride=n, g_stride=0 if shared_g else n, y_stride=n)
    D = Q.trunc(*dec)
    F = Q.trunc(*fft)
    nb = Q.qtt_workspace_bytes(shp, D, F)
    w = ws(nb)
    y = torch.empty(f.size, dtype=torch.float64, device="cuda")
    rep = Q.qtt_conv_full(fd.data_ptr(), gd.data_ptr(), y.data_ptr(), shp, D, F, shift, scale,
                          w.data_ptr(), nb, stream(), report=report)
    torch.cuda.synchronize()
    return y.cpu().numpy().reshape(f.shape), rep


def gpu_tt_from_cores(cores_list, like, layout, rcap=10):
    """Upload (oracle) cores as a GPU TT handle (test-only entry point)."""
    d = len(cores_list)
    buf = np.zeros(d * 512, np.complex128)
    ranks = np.zeros(64, np.int32)
    ranks[0] = 1
    for k, c in enumerate(cores_list):
        buf[k * 512: k * 512 + c.size] = np.asarray(c, np.complex128).reshape(-1, order="F")
        ranks[k + 1] = c.shape[2]
    shp = shape_of(like, layout)
    w = ws(d * 512 * 16 + 1 << 16)
    return Q.qtt_debug_tt_from_host(shp, buf, ranks, rcap, w.data_ptr(), w.numel() - 256, stream(),
                                    ws_owner=w)
