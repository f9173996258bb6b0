"""Host logic of the column-sharded path (no GPU): the library's shard
geometry (qtt_shard_geometry) against the definition in include/qtt.h /
SURVEY §8(e) — shard s holds exactly the QTT indices whose top l bits equal
s, stored as a dense row-major sub-image in the shard's own (local) QTT
layout — plus communicator and workspace validation."""

import ctypes

import numpy as np
import pytest

import oracle as O
from paper_2301_13339_b200 import build as B
from paper_2301_13339_b200 import qtt as Q
from paper_2301_13339_b200 import shard as SH


@pytest.fixture(scope="module", autouse=True)
def L():
    B.build()
    return Q.lib()


def _compact_even(q):
    out = np.zeros_like(q)
    for t in range(31):
        out |= ((q >> (2 * t)) & 1) << t
    return out


def _global_xy(q, D, b, layout):
    """Grid point of global QTT index q (definition, P:298-307 / reading Q8)."""
    if D == 1:
        return q, np.zeros_like(q)
    if layout == "interleaved":
        return _compact_even(q), _compact_even(q >> 1)
    return q & ((1 << b) - 1), q >> b          # concat: x bits, then y bits


def _local_xy(q, D, bits, layout):
    """Grid point of local QTT index q inside a (possibly rectangular) shard."""
    if D == 1:
        return q, np.zeros_like(q)
    if layout == "interleaved":
        return _compact_even(q), _compact_even(q >> 1)   # x takes the extra (top) bit
    return q & ((1 << bits[0]) - 1), q >> bits[0]


CASES = [(1, 15, "1d"), (2, 7, "interleaved"), (2, 8, "interleaved"), (2, 8, "concat")]


@pytest.mark.parametrize("D,b,layout", CASES)
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_shard_geometry_is_the_top_bit_range(D, b, layout, P):
    shp = Q.shape(D, [b, b], layout)
    d = D * b
    if d - int(np.log2(P)) < 12:
        pytest.skip("shard below the 2^12 minimum")
    l = int(np.log2(P))
    dl = d - l
    seen = np.zeros((1 << b,) * D, dtype=np.int32)
    for s in range(P):
        (x0, y0), bits = Q.qtt_shard_geometry(shp, P, s)
        assert (1 << bits[0]) * (1 << bits[1] if D == 2 else 1) == 1 << dl
        if layout == "interleaved":
            assert bits == ((dl + 1) // 2, dl // 2)
        q = np.arange(1 << dl, dtype=np.int64)
        gx, gy = _global_xy((s << dl) + q, D, b, layout)     # top l bits = s
        lx, ly = _local_xy(q, D, bits, layout)
        np.testing.assert_array_equal(gx, x0 + lx)
        np.testing.assert_array_equal(gy, y0 + ly)
        if D == 1:
            seen[x0:x0 + (1 << bits[0])] += 1
        else:
            seen[y0:y0 + (1 << bits[1]), x0:x0 + (1 << bits[0])] += 1
    assert (seen == 1).all()          # a partition of the array


def test_shard_local_qtt_order_matches_oracle_on_square_shards():
    """For P = 4 interleaved shards are square, so the oracle's to_qtt of a
    shard must equal the corresponding slice of the global QTT vector."""
    b = 7
    shp = Q.shape(2, [b, b], "interleaved")
    x = np.random.default_rng(0).standard_normal((1 << b, 1 << b))
    v = O.to_qtt(x, "interleaved")
    P, dl = 4, 2 * b - 2
    for s, part in enumerate(SH.split(x, shp, P)):
        np.testing.assert_array_equal(O.to_qtt(np.ascontiguousarray(part), "interleaved"),
                                      v[s << dl:(s + 1) << dl])


def test_split_assemble_roundtrip():
    shp = Q.shape(2, [8, 8], "interleaved")
    x = np.arange(1 << 16, dtype=np.float64).reshape(256, 256)
    for P in (2, 4, 8):
        parts = [np.ascontiguousarray(p) for p in SH.split(x, shp, P)]
        out = SH.assemble(parts, shp, P, np.zeros_like(x))
        np.testing.assert_array_equal(out, x)


def test_shard_geometry_rejects_bad_requests():
    o = (ctypes.c_longlong * 2)()
    bb = (ctypes.c_int * 2)()
    L = Q.lib()
    shp = Q.shape(2, [7, 7], "interleaved")
    assert L.qtt_shard_geometry(ctypes.byref(shp), 3, 0, o, bb) == Q.QTT_EINVAL      # not 2^l
    assert L.qtt_shard_geometry(ctypes.byref(shp), 4, 4, o, bb) == Q.QTT_EINVAL      # shard index
    assert L.qtt_shard_geometry(ctypes.byref(shp), 8, 0, o, bb) == Q.QTT_EINVAL      # d - l = 11 < 12
    assert b"shard must hold" in L.qtt_last_error()
    small = Q.shape(2, [6, 6], "concat")
    assert L.qtt_shard_geometry(ctypes.byref(small), 2, 0, o, bb) == Q.QTT_EINVAL


def test_comm_virtual_and_workspace():
    dec, fft = Q.trunc(1e-3, 10), Q.trunc(1e-3, 8)
    shp = Q.shape(2, [9, 9], "interleaved")
    big = Q.shape(2, [12, 12], "interleaved")
    one = Q.qtt_workspace_bytes(big, dec, fft, 1)
    n2 = Q.qtt_workspace_bytes(big, dec, fft, 2)
    n8 = Q.qtt_workspace_bytes(big, dec, fft, 8)
    assert 0 < n8 < n2 < one          # per-rank unfolding scratch shrinks with P
    c = Q.qtt_comm_init_virtual(4)
    nv = Q.qtt_comm_workspace_bytes(shp, dec, fft, c)
    assert nv > Q.qtt_workspace_bytes(shp, dec, fft, 4)   # all 4 shards in one process
    c.close()
    h = ctypes.c_void_p()
    assert Q.lib().qtt_comm_init_virtual(3, ctypes.byref(h)) == Q.QTT_EINVAL
    # sharding needs batch 1, and a dec cap the all-gather supports
    c = Q.qtt_comm_init_virtual(2)
    with pytest.raises(Q.QttError):
        Q.qtt_comm_workspace_bytes(Q.shape(2, [9, 9], "interleaved", batch=2), dec, fft, c)
    c.close()
