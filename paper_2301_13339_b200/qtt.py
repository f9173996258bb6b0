"""Thin ctypes binding of libqtt.so (include/qtt.h).

Argument marshalling only: every step of the QTT convolution runs in the
library's sm_100a kernels.  Device pointers are plain integers (e.g.
`torch.Tensor.data_ptr()`), streams are `cudaStream_t` integers (e.g.
`torch.cuda.current_stream().cuda_stream`).  There is no CPU fallback: if the
library is missing, `lib()` raises.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QTT_LIB", os.path.join(HERE, "libqtt.so"))   # override: diagnostics builds

QTT_OK, QTT_EINVAL, QTT_ENUMERIC, QTT_ECUDA, QTT_ENCCL, QTT_ENOMEM = range(6)
LAYOUTS = {"1d": 0, "interleaved": 1, "concat": 2}

SYMBOLS = [
    "qtt_workspace_bytes", "qtt_decompose", "qtt_transform", "qtt_convolve",
    "qtt_to_full", "qtt_conv_full", "qtt_wait", "qtt_ranks", "qtt_ndims",
    "qtt_destroy", "qtt_status_string", "qtt_last_error", "qtt_build_info",
    "qtt_debug_eigh", "qtt_debug_tt_from_host", "qtt_profile_enable", "qtt_profile_read",
    "qtt_launch_count", "qtt_comm_workspace_bytes", "qtt_comm_unique_id", "qtt_comm_init",
    "qtt_comm_init_virtual", "qtt_comm_destroy", "qtt_shard_geometry", "qtt_debug_omega",
]


class Shape(ctypes.Structure):
    _fields_ = [("D", ctypes.c_int), ("bits", ctypes.c_int * 2), ("layout", ctypes.c_int),
                ("batch", ctypes.c_int), ("f_stride", ctypes.c_longlong),
                ("g_stride", ctypes.c_longlong), ("y_stride", ctypes.c_longlong)]


class Trunc(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("rmax", ctypes.c_int), ("cluster_tol", ctypes.c_double),
                ("rule", ctypes.c_int), ("delta", ctypes.c_double), ("p", ctypes.c_int),
                ("seed", ctypes.c_ulonglong)]


class Report(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("ranks_f", ctypes.c_int * 64), ("ranks_g", ctypes.c_int * 64),
                ("ranks_fh", ctypes.c_int * 64), ("ranks_gh", ctypes.c_int * 64),
                ("ranks_z", ctypes.c_int * 64), ("ranks_out", ctypes.c_int * 64),
                ("ms_total", ctypes.c_float), ("status_bits", ctypes.c_int),
                ("min_margin", ctypes.c_double), ("min_gap", ctypes.c_double)]


class QttError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} (status {status})")
        self.status = status


_LIB = None


def lib():
    """Load libqtt.so (raises if it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: build it with __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    P, I, S, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_double
    pS, pT, pH = ctypes.POINTER(Shape), ctypes.POINTER(Trunc), ctypes.POINTER(ctypes.c_void_p)
    pLL = ctypes.POINTER(ctypes.c_longlong)
    L.qtt_workspace_bytes.restype = S
    L.qtt_workspace_bytes.argtypes = [pS, pT, pT, I]
    L.qtt_decompose.restype = I
    L.qtt_decompose.argtypes = [P, pS, pT, P, S, P, P, pH]
    L.qtt_transform.restype = I
    L.qtt_transform.argtypes = [P, pT, I, pLL, D, P, S, P, pH]
    L.qtt_convolve.restype = I
    L.qtt_convolve.argtypes = [P, P, pT, pLL, D, P, S, P, pH]
    L.qtt_to_full.restype = I
    L.qtt_to_full.argtypes = [P, P, P, P, S, P, P]
    L.qtt_conv_full.restype = I
    L.qtt_conv_full.argtypes = [P, P, P, pS, pT, pT, pLL, D, P, S, P, P, ctypes.POINTER(Report)]
    L.qtt_wait.restype = I
    L.qtt_wait.argtypes = [P]
    L.qtt_ranks.restype = I
    L.qtt_ranks.argtypes = [P, I, ctypes.POINTER(ctypes.c_int), I]
    L.qtt_ndims.restype = I
    L.qtt_ndims.argtypes = [P]
    L.qtt_destroy.restype = None
    L.qtt_destroy.argtypes = [P]
    L.qtt_status_string.restype = ctypes.c_char_p
    L.qtt_status_string.argtypes = [I]
    L.qtt_last_error.restype = ctypes.c_char_p
    L.qtt_last_error.argtypes = []
    L.qtt_build_info.restype = ctypes.c_char_p
    L.qtt_build_info.argtypes = []
    L.qtt_debug_eigh.restype = I
    L.qtt_debug_eigh.argtypes = [P, I, P, P, P, I, I, P]
    L.qtt_profile_enable.restype = None
    L.qtt_profile_enable.argtypes = [I]
    L.qtt_profile_read.restype = I
    L.qtt_profile_read.argtypes = [ctypes.POINTER(ctypes.c_float), I]
    L.qtt_launch_count.restype = ctypes.c_longlong
    L.qtt_launch_count.argtypes = []
    L.qtt_comm_workspace_bytes.restype = S
    L.qtt_comm_workspace_bytes.argtypes = [pS, pT, pT, P]
    L.qtt_comm_unique_id.restype = I
    L.qtt_comm_unique_id.argtypes = [ctypes.c_char_p]
    L.qtt_comm_init.restype = I
    L.qtt_comm_init.argtypes = [ctypes.c_char_p, I, I, pH]
    L.qtt_comm_init_virtual.restype = I
    L.qtt_comm_init_virtual.argtypes = [I, pH]
    L.qtt_comm_destroy.restype = None
    L.qtt_comm_destroy.argtypes = [P]
    L.qtt_shard_geometry.restype = I
    L.qtt_shard_geometry.argtypes = [pS, I, I, pLL, ctypes.POINTER(ctypes.c_int)]
    L.qtt_debug_omega.restype = I
    L.qtt_debug_omega.argtypes = [ctypes.c_ulonglong, I, ctypes.c_ulonglong, I, I, P, P]
    L.qtt_debug_tt_from_host.restype = I
    L.qtt_debug_tt_from_host.argtypes = [pS, P, ctypes.POINTER(ctypes.c_int), I, P, S, P, pH]
    _LIB = L
    return L


def _check(st):
    if st != QTT_OK:
        L = lib()
        raise QttError(st, f"{L.qtt_status_string(st).decode()}: {L.qtt_last_error().decode()}")


def shape(D, bits, layout="1d", batch=1, f_stride=0, g_stride=0, y_stride=0):
    b = (ctypes.c_int * 2)(bits[0], bits[1] if D == 2 else 0)
    return Shape(D, b, LAYOUTS[layout], batch, f_stride, g_stride, y_stride)


def trunc(eps, rmax, cluster_tol=1e-10, delta=None, rsvd=None):
    """Truncation policy: RANK(eps, rmax, cluster_tol) (modification (1));
    with `delta` the SV drop-off rule (modification (3)) capped at rmax; with
    rsvd = (p, seed) the max-rank TT-RSVD (modification (2), decomposition
    only)."""
    if rsvd is not None:
        return Trunc(eps, rmax, cluster_tol, 2, 0.0, int(rsvd[0]), int(rsvd[1]))
    if delta is None:
        return Trunc(eps, rmax, cluster_tol, 0, 0.0, 0, 0)
    return Trunc(eps, rmax, cluster_tol, 1, float(delta), 0, 0)


def _shift(shift):
    if shift is None:
        return None
    s = list(shift) + [0] * (2 - len(shift))
    return (ctypes.c_longlong * 2)(*s)


class TT:
    """Owning wrapper of a qtt_tt_t handle (device storage lives in `ws`)."""

    def __init__(self, handle, ws=None):
        self.h = handle
        self.ws = ws            # keep the workspace alive

    def ranks(self, index=0):
        d = lib().qtt_ndims(self.h)
        buf = (ctypes.c_int * (d + 1))()
        _check(lib().qtt_ranks(self.h, index, buf, d + 1))
        return list(buf)

    def wait(self):
        _check(lib().qtt_wait(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.qtt_destroy(self.h)
            self.h = None


def qtt_workspace_bytes(shp, dec, fft, nranks=1):
    n = lib().qtt_workspace_bytes(ctypes.byref(shp), ctypes.byref(dec), ctypes.byref(fft), nranks)
    if n == 0:
        raise QttError(QTT_EINVAL, "invalid shape / truncation for qtt_workspace_bytes")
    return n


def qtt_decompose(x_ptr, shp, dec, ws_ptr, ws_bytes, stream=0, ws_owner=None, comm=None):
    h = ctypes.c_void_p()
    _check(lib().qtt_decompose(x_ptr, ctypes.byref(shp), ctypes.byref(dec), ws_ptr, ws_bytes,
                               stream, _comm(comm), ctypes.byref(h)))
    return TT(h, ws_owner)


def qtt_transform(tt, fft, inverse, shift, scale, ws_ptr, ws_bytes, stream=0, ws_owner=None):
    h = ctypes.c_void_p()
    _check(lib().qtt_transform(tt.h, ctypes.byref(fft), int(inverse), _shift(shift), float(scale),
                               ws_ptr, ws_bytes, stream, ctypes.byref(h)))
    return TT(h, ws_owner)


def qtt_convolve(f, g, fft, shift, scale, ws_ptr, ws_bytes, stream=0, ws_owner=None):
    h = ctypes.c_void_p()
    _check(lib().qtt_convolve(f.h, g.h, ctypes.byref(fft), _shift(shift), float(scale), ws_ptr,
                              ws_bytes, stream, ctypes.byref(h)))
    return TT(h, ws_owner)


def qtt_to_full(tt, y_ptr, ws_ptr, ws_bytes, stream=0, y_imag_ptr=None, comm=None):
    _check(lib().qtt_to_full(tt.h, y_ptr, y_imag_ptr, ws_ptr, ws_bytes, stream, _comm(comm)))


def qtt_conv_full(f_ptr, g_ptr, y_ptr, shp, dec, fft, shift, scale, ws_ptr, ws_bytes, stream=0,
                  report=False, comm=None):
    rep = Report() if report else None
    _check(lib().qtt_conv_full(f_ptr, g_ptr, y_ptr, ctypes.byref(shp), ctypes.byref(dec),
                               ctypes.byref(fft), _shift(shift), float(scale), ws_ptr, ws_bytes,
                               stream, _comm(comm), ctypes.byref(rep) if rep is not None else None))
    if rep is None:
        return None
    d = rep.d
    return {"d": d, "ranks_f": list(rep.ranks_f[:d + 1]), "ranks_g": list(rep.ranks_g[:d + 1]),
            "ranks_fh": list(rep.ranks_fh[:d + 1]), "ranks_gh": list(rep.ranks_gh[:d + 1]),
            "ranks_z": list(rep.ranks_z[:d + 1]), "ranks_out": list(rep.ranks_out[:d + 1]),
            "ms_total": rep.ms_total, "status_bits": rep.status_bits,
            "min_margin": rep.min_margin, "min_gap": rep.min_gap}


class Comm:
    """Owning wrapper of a qtt_comm_t (NCCL or virtual shards)."""

    def __init__(self, handle, nshards, nlocal, first):
        self.h = handle
        self.nshards = nshards      # P
        self.nlocal = nlocal        # shards held by this process
        self.first = first          # index of this process's first shard

    def close(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.qtt_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def _comm(comm):
    return None if comm is None else comm.h


def qtt_comm_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(lib().qtt_comm_unique_id(buf))
    return buf.raw


def qtt_comm_init(uid, nranks, rank):
    """NCCL communicator; `uid` = rank 0's qtt_comm_unique_id() bytes."""
    h = ctypes.c_void_p()
    _check(lib().qtt_comm_init(bytes(uid), nranks, rank, ctypes.byref(h)))
    return Comm(h, nranks, 1, rank)


def qtt_comm_init_virtual(nshards):
    h = ctypes.c_void_p()
    _check(lib().qtt_comm_init_virtual(nshards, ctypes.byref(h)))
    return Comm(h, nshards, nshards, 0)


def qtt_comm_workspace_bytes(shp, dec, fft, comm):
    n = lib().qtt_comm_workspace_bytes(ctypes.byref(shp), ctypes.byref(dec), ctypes.byref(fft),
                                       _comm(comm))
    if n == 0:
        raise QttError(QTT_EINVAL, "invalid shape / truncation / sharding")
    return n


def qtt_shard_geometry(shp, nshards, shard):
    """(origin (x0, y0), bits (bx, by)) of a shard in the global array."""
    o = (ctypes.c_longlong * 2)()
    b = (ctypes.c_int * 2)()
    _check(lib().qtt_shard_geometry(ctypes.byref(shp), nshards, shard, o, b))
    return (int(o[0]), int(o[1])), (int(b[0]), int(b[1]))


def build_info():
    return lib().qtt_build_info().decode()


def qtt_debug_eigh(a_ptr, n, lam_ptr, u_ptr, sweeps_ptr, stream=0, reps=1, mode=0):
    """Test-only: the path's small Hermitian eigensolver on one matrix
    (mode 0: tridiagonal with Jacobi fallback, as in production; 1: Jacobi)."""
    _check(lib().qtt_debug_eigh(a_ptr, n, lam_ptr, u_ptr, sweeps_ptr, reps, mode, stream))


def qtt_debug_tt_from_host(shp, cores_c128, ranks_i32, rcap, ws_ptr, ws_bytes, stream=0, ws_owner=None):
    """Test-only: upload cores (complex128 array of nt*d*512) and ranks (int32 nt*64)."""
    h = ctypes.c_void_p()
    _check(lib().qtt_debug_tt_from_host(ctypes.byref(shp), cores_c128.ctypes.data,
                                        ranks_i32.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                        rcap, ws_ptr, ws_bytes, stream, ctypes.byref(h)))
    return TT(h, ws_owner)


def qtt_debug_omega(seed, k, j0, n, kp, out_ptr, stream=0):
    """Test-only: Omega_k rows j0..j0+n-1 (row-major n x kp) on the device."""
    _check(lib().qtt_debug_omega(seed, k, j0, n, kp, out_ptr, stream))


STAGES = ["ttsvd", "qfft", "hadamard_round", "qifft", "expand"]


def qtt_profile_enable(on=True):
    """on: False/0 off, True/1 stage events, 2 stage + full-array pass events
    (the decomposition then runs as one chain on the caller's stream)."""
    lib().qtt_profile_enable(int(on))


PASSES = ("pass_level_gram", "pass_project_x", "pass_project_w", "pass_expand")


def qtt_profile_read():
    buf = (ctypes.c_float * 16)()
    n = lib().qtt_profile_read(buf, 16)
    out = {STAGES[i]: float(buf[i]) for i in range(min(n, len(STAGES)))}
    for i in range(len(STAGES), n):
        if buf[i] >= 0:
            out[PASSES[i - len(STAGES)]] = float(buf[i])
    return out


def qtt_launch_count():
    return int(lib().qtt_launch_count())
