"""GPU parity of the column-sharded path (include/qtt.h "Multi-GPU", SURVEY
§8(e)) through the C ABI.

One GPU cannot host ranks that wait on each other, so the sharded kernels are
exercised two ways: (1) a virtual communicator — all P shards in this process,
the cross-shard Gram sums done by a kernel — for P = 1, 2, 4, 8; (2) a real
NCCL communicator of one rank (the collectives run, trivially).  Both are
compared with the unsharded float64 oracle: identical ranks, rel-L2 <= 1e-9
(north star)."""

import numpy as np
import pytest
import torch

import oracle as O
from paper_2301_13339_b200 import qtt as Q
from paper_2301_13339_b200 import shard as SH
from paper_2301_13339_b200 import synth

from gpu_util import dev, gpu_decompose, gpu_full, shape_of, stream, ws

pytestmark = pytest.mark.gpu

TOL = 1e-9


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _stack(x, shp, P):
    return np.concatenate([np.ascontiguousarray(p).reshape(-1) for p in SH.split(x, shp, P)])


def _unstack(y, shp, P, like):
    n = like.size // P
    parts = [y[j * n:(j + 1) * n] for j in range(P)]
    return SH.assemble(parts, shp, P, np.zeros_like(like))


def sharded_conv(f, g, layout, dec, fft, shift, scale, comm):
    shp = shape_of(f, layout)
    P = comm.nshards
    fd, gd = dev(_stack(f, shp, P)), dev(_stack(g, shp, P))
    D, F = Q.trunc(*dec), Q.trunc(*fft)
    nb = Q.qtt_comm_workspace_bytes(shp, D, F, comm)
    w = ws(nb)
    y = torch.empty_like(fd)
    rep = Q.qtt_conv_full(fd.data_ptr(), gd.data_ptr(), y.data_ptr(), shp, D, F, shift, scale,
                          w.data_ptr(), nb, stream(), report=True, comm=comm)
    torch.cuda.synchronize()
    return _unstack(y.cpu().numpy(), shp, P, f), rep


_REF = {}


def oracle_conv(name):
    if name not in _REF:
        if name == "c2":
            p = synth.problem("c2")
            f, g = synth.signal("c2"), synth.kernel(2, 9, 60.0)
            lay, eps = "interleaved", p["eps"][0]
            shift, scale = p["shift"], p["scale"]
        elif name == "1d16":
            f = synth.random_signal((1 << 16,), 21)
            g = synth.kernel(1, 16, 300.0)
            lay, eps, shift, scale = "1d", 1e-3, (1 << 15,), 2.0 / (1 << 16)
        else:   # concat 256 x 256
            f = synth.random_signal((256, 256), 22, "smooth")
            g = synth.kernel(2, 8, 40.0)
            lay, eps, shift, scale = "concat", 1e-4, (128, 128), (2.0 / 256) ** 2
        dec, fft = (eps, 10, 1e-10), (eps, 8, 1e-10)
        want, info = O.conv_pipeline(f, g, lay, dec, fft, shift, scale, return_info=True)
        _REF[name] = (f, g, lay, dec, fft, shift, scale, want, info)
    return _REF[name]


@pytest.mark.parametrize("name,P", [("c2", 1), ("c2", 2), ("c2", 4), ("c2", 8),
                                    ("1d16", 2), ("1d16", 8), ("concat", 4)])
def test_virtual_sharded_conv_matches_oracle(name, P):
    f, g, lay, dec, fft, shift, scale, want, info = oracle_conv(name)
    comm = Q.qtt_comm_init_virtual(P)
    y, rep = sharded_conv(f, g, lay, dec, fft, shift, scale, comm)
    comm.close()
    assert rep["status_bits"] & 3 == 0
    assert rep["ranks_f"] == O.ranks_of(info["F"])
    assert rep["ranks_g"] == O.ranks_of(info["G"])
    assert rep["ranks_out"] == O.ranks_of(info["Y"])
    assert rel(y, want) <= TOL


def test_nccl_one_rank_conv_matches_oracle():
    f, g, lay, dec, fft, shift, scale, want, info = oracle_conv("c2")
    comm = Q.qtt_comm_init(Q.qtt_comm_unique_id(), 1, 0)
    y, rep = sharded_conv(f, g, lay, dec, fft, shift, scale, comm)
    comm.close()
    assert rep["ranks_out"] == O.ranks_of(info["Y"])
    assert rel(y, want) <= TOL


@pytest.mark.parametrize("P", [2, 8])
def test_virtual_sharded_decompose_and_expand(P):
    """Sharded TT-SVD -> unsharded expansion, and unsharded TT-SVD -> sharded
    expansion, both against the oracle's TT-SVD."""
    x = synth.random_signal((512, 512), 23, "smooth")
    eps = 1e-5
    ref = O.tt_svd(O.to_qtt(x, "interleaved"), eps, 10, 1e-10)
    want = O.from_qtt(O.full(ref), x.shape, "interleaved")
    shp = shape_of(x, "interleaved")
    dec = Q.trunc(eps, 10, 1e-10)
    comm = Q.qtt_comm_init_virtual(P)
    nb = Q.qtt_comm_workspace_bytes(shp, dec, Q.trunc(eps, 8), comm)
    w = ws(nb)
    xd = dev(_stack(x, shp, P))
    tt = Q.qtt_decompose(xd.data_ptr(), shp, dec, w.data_ptr(), nb, stream(), ws_owner=w, comm=comm)
    assert tt.ranks() == O.ranks_of(ref)
    assert rel(gpu_full(tt, x), want) <= TOL
    # unsharded decomposition, sharded expansion
    tt2 = gpu_decompose(x, "interleaved", eps, 10)
    y = torch.empty(x.size, dtype=torch.float64, device="cuda")
    w2 = ws(1 << 24)
    Q.qtt_to_full(tt2, y.data_ptr(), w2.data_ptr(), 1 << 24, stream(), comm=comm)
    torch.cuda.synchronize()
    assert rel(_unstack(y.cpu().numpy(), shp, P, x), want) <= TOL
    comm.close()


def test_sharded_rejects_batch_and_small_shards():
    x = synth.random_signal((64, 64), 1)
    shp = shape_of(x, "interleaved")
    comm = Q.qtt_comm_init_virtual(2)         # d = 12 -> shards of 2^11 < 2^12
    w = ws(1 << 24)
    xd = dev(x)
    with pytest.raises(Q.QttError) as e:
        Q.qtt_decompose(xd.data_ptr(), shp, Q.trunc(1e-3, 10), w.data_ptr(), 1 << 24, stream(),
                        comm=comm)
    assert e.value.status == Q.QTT_EINVAL
    comm.close()
