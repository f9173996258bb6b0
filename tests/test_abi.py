"""The C-ABI library (no GPU needed): it loads, exports every function
include/qtt.h declares, and its host-side validation and workspace sizing
behave as documented."""

import ctypes
import os
import re

import pytest

from paper_2301_13339_b200 import build as B
from paper_2301_13339_b200 import qtt as Q

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    B.build()
    return Q.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "qtt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qtt_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n
    assert sorted(Q.SYMBOLS) == names


def test_build_info_names_sm100a(L):
    assert "sm_100a" in Q.build_info()


def test_status_strings(L):
    assert L.qtt_status_string(0) == b"QTT_OK"
    assert L.qtt_status_string(1) == b"QTT_EINVAL"
    assert L.qtt_status_string(5) == b"QTT_ENOMEM"


def test_workspace_bytes_validation(L):
    dec, fft = Q.trunc(1e-3, 10), Q.trunc(1e-3, 8)
    n18 = Q.qtt_workspace_bytes(Q.shape(2, [9, 9], "interleaved"), dec, fft)
    n20 = Q.qtt_workspace_bytes(Q.shape(2, [10, 10], "interleaved"), dec, fft)
    assert 0 < n18 < n20
    # batch with a shared kernel grows the plan
    nb = Q.qtt_workspace_bytes(Q.shape(2, [9, 9], "interleaved", batch=4), dec, fft)
    assert nb > n18
    bad = [
        (Q.shape(3, [9, 9]), dec, fft),                          # D
        (Q.shape(2, [9, 8], "interleaved"), dec, fft),            # non-square interleave
        (Q.shape(1, [40, 0]), dec, fft),                          # d > 30
        (Q.shape(1, [1, 0]), dec, fft),                           # d < 2
        (Q.shape(2, [9, 9], "1d"), dec, fft),                     # layout mismatch
        (Q.shape(2, [9, 9], "interleaved"), Q.trunc(-1.0, 10), fft),
        (Q.shape(2, [9, 9], "interleaved"), Q.trunc(1e-3, 0), fft),
        (Q.shape(2, [9, 9], "interleaved"), dec, Q.trunc(1e-3, 17)),  # Rhat > 16
        (Q.shape(2, [9, 9], "interleaved"), Q.trunc(1e-3, 17), fft),  # R_max > 16
    ]
    for s, a, b in bad:
        assert L.qtt_workspace_bytes(ctypes.byref(s), ctypes.byref(a), ctypes.byref(b), 1) == 0
    # the paper's caps (10, 15) and (16, 16) are valid; sharded plans keep R_max <= 10
    shp = Q.shape(2, [9, 9], "interleaved")
    for a, b in ((dec, Q.trunc(1e-3, 15)), (Q.trunc(1e-3, 16), Q.trunc(1e-3, 16))):
        assert L.qtt_workspace_bytes(ctypes.byref(shp), ctypes.byref(a), ctypes.byref(b), 1) > 0
    big = Q.trunc(1e-3, 16)
    assert L.qtt_workspace_bytes(ctypes.byref(shp), ctypes.byref(big), ctypes.byref(fft), 2) == 0


def test_invalid_arguments_fail_before_any_device_work(L):
    h = ctypes.c_void_p()
    s = Q.shape(3, [9, 9])
    st = L.qtt_decompose(None, ctypes.byref(s), ctypes.byref(Q.trunc(1e-3, 10)), None, 0, None,
                         None, ctypes.byref(h))
    assert st == Q.QTT_EINVAL
    assert b"D must be" in L.qtt_last_error()
    s = Q.shape(1, [12, 0])
    st = L.qtt_conv_full(None, None, None, ctypes.byref(s), ctypes.byref(Q.trunc(1e-3, 10)),
                         ctypes.byref(Q.trunc(1e-3, 8)), None, 1.0, None, 0, None, None, None)
    assert st == Q.QTT_EINVAL
    # workspace too small is reported as ENOMEM, not a device fault
    st = L.qtt_conv_full(ctypes.c_void_p(256), ctypes.c_void_p(256), ctypes.c_void_p(256),
                         ctypes.byref(s), ctypes.byref(Q.trunc(1e-3, 10)),
                         ctypes.byref(Q.trunc(1e-3, 8)), None, 1.0, ctypes.c_void_p(256), 1024,
                         None, None, None)
    assert st == Q.QTT_ENOMEM


def test_truncation_rule_validation(L):
    shp = Q.shape(2, [9, 9], "interleaved")
    fft = Q.trunc(1e-3, 8)
    ok = Q.trunc(0.0, 10, 1e-10, delta=0.02)
    assert ok.rule == 1 and ok.delta == 0.02
    assert L.qtt_workspace_bytes(ctypes.byref(shp), ctypes.byref(ok), ctypes.byref(fft), 1) > 0
    for bad in (Q.Trunc(0.0, 10, 1e-10, 1, 0.0), Q.Trunc(0.0, 10, 1e-10, 1, 1.0), Q.Trunc(1e-3, 10, 1e-10, 7, 0.1)):
        assert L.qtt_workspace_bytes(ctypes.byref(shp), ctypes.byref(bad), ctypes.byref(fft), 1) == 0


def test_misaligned_inputs_are_rejected_before_device_work(L):
    """The TT-SVD streams f / g / x with 16-byte copies: a misaligned input
    or an odd batch stride is QTT_EINVAL, never a sticky device fault
    (ADVICE r1)."""
    s = Q.shape(1, [14, 0])
    dec, fft = Q.trunc(1e-3, 10), Q.trunc(1e-3, 8)
    nb = L.qtt_workspace_bytes(ctypes.byref(s), ctypes.byref(dec), ctypes.byref(fft), 1)
    ws = ctypes.c_void_p(1 << 20)
    ok, bad = ctypes.c_void_p(4096), ctypes.c_void_p(4096 + 8)
    for f, g in ((bad, ok), (ok, bad)):
        st = L.qtt_conv_full(f, g, ok, ctypes.byref(s), ctypes.byref(dec), ctypes.byref(fft), None, 1.0,
                             ws, nb, None, None, None)
        assert st == Q.QTT_EINVAL and b"16-byte aligned" in L.qtt_last_error()
    h = ctypes.c_void_p()
    st = L.qtt_decompose(bad, ctypes.byref(s), ctypes.byref(dec), ws, nb, None, None, ctypes.byref(h))
    assert st == Q.QTT_EINVAL
    sb = Q.shape(1, [14, 0], "1d", 2, (1 << 14) + 1, 0, 0)
    nbb = L.qtt_workspace_bytes(ctypes.byref(sb), ctypes.byref(dec), ctypes.byref(fft), 1)
    st = L.qtt_decompose(ok, ctypes.byref(sb), ctypes.byref(dec), ws, nbb, None, None, ctypes.byref(h))
    assert st == Q.QTT_EINVAL and b"stride must be even" in L.qtt_last_error()
