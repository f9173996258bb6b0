"""The column-sharded algorithm of the multi-GPU path (include/qtt.h
"Multi-GPU") on CPU with world_size 2 over gloo.

Each rank takes its shard of a seeded global array, placed by the library's
own qtt_shard_geometry (host logic of the GPU path), and runs the same
sequence the GPU driver (api.cu run_sharded_dec / run_sharded_expand)
launches, written in numpy:
  * Alg. 1 steps k while the local unfolding is wide: local Gram, ALLREDUCE,
    eigendecomposition + RANK, local projection;
  * ALL-GATHER of the narrow remainder W, remaining steps redundantly;
  * expansion of the rank's shard by folding the top l cores at the shard's
    bits (Alg. 3).
It checks the result against the unsharded oracle (oracle.tt_svd / full):
identical ranks, reconstruction and shard of the expansion to rounding."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2301_13339_b200 import build as B
from paper_2301_13339_b200 import qtt as Q
from paper_2301_13339_b200 import shard as SH
from paper_2301_13339_b200 import synth


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _compact_even(q):
    out = np.zeros_like(q)
    for t in range(31):
        out |= ((q >> (2 * t)) & 1) << t
    return out


def _local_qtt(part, D, bits, layout):
    """A shard's values in its local QTT order."""
    if D == 1 or layout == "concat":
        return np.ascontiguousarray(part).reshape(-1)
    q = np.arange(part.size, dtype=np.int64)
    return part[_compact_even(q >> 1), _compact_even(q)]


def _allreduce(a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _allgather_cols(W):
    t = torch.from_numpy(np.ascontiguousarray(W))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.concatenate([o.numpy() for o in out], axis=1)


def _step(M, tau2, rmax, ctol, d, k, reduce):
    G = M @ M.T
    if reduce:
        G = _allreduce(G)
    lam, U = np.linalg.eigh(G)
    lam, U = lam[::-1], U[:, ::-1]
    mp_ = min(M.shape[0], 1 << (d - k))
    r = O.rank_rule(lam[:mp_], tau2, rmax, ctol)
    return U[:, :r], r


def sharded_tt_svd(v_loc, d, dl, eps, rmax, ctol):
    """Mirror of run_sharded_dec: returns the global cores on every rank."""
    tau2 = eps * eps * float(_allreduce(np.array([v_loc @ v_loc]))[0]) / (d - 1)
    cores, r, W, k = [], 1, v_loc.reshape(1, -1), 1
    # level stage (steps 1..5) and then while the local W_{k-1} has >= 256 columns
    while k <= d - 1 and (k <= 5 or ((1 << (dl - k + 1)) >= 256 and (1 << (d - k + 1)) > 256)):
        M = W.reshape(2 * r, -1, order="F")
        U, rk = _step(M, tau2, rmax, ctol, d, k, True)
        cores.append(U.reshape(r, 2, rk, order="F"))
        W, r, k = U.T @ M, rk, k + 1
    W = _allgather_cols(W)              # shard-major columns = global column order
    while k <= d - 1:
        M = W.reshape(2 * r, -1, order="F")
        U, rk = _step(M, tau2, rmax, ctol, d, k, False)
        cores.append(U.reshape(r, 2, rk, order="F"))
        W, r, k = U.T @ M, rk, k + 1
    cores.append(W.reshape(r, 2, 1, order="F"))
    return cores


def fold_tail(cores, l, shard):
    """Mirror of k_fold_tail: cores of the shard whose top l bits are `shard`."""
    d = len(cores)
    v = np.ones(1)
    for k in range(d, d - l, -1):
        bit = (shard >> (k - (d - l) - 1)) & 1
        v = cores[k - 1][:, bit, :] @ v
    last = np.einsum("aib,b->ai", cores[d - l - 1], v)[:, :, None]
    return cores[:d - l - 1] + [last]


CASES = {
    "2d_lowrank": dict(D=2, b=8, layout="interleaved", kind="lowrank", eps=1e-5, seed=11),
    "2d_c2": dict(D=2, b=9, layout="interleaved", kind="c2", eps=1e-3, seed=0),
    "1d_smooth": dict(D=1, b=15, layout="1d", kind="smooth", eps=1e-6, seed=12),
    "2d_concat": dict(D=2, b=8, layout="concat", kind="lowrank", eps=1e-5, seed=13),
}


def _global(c):
    if c["kind"] == "c2":
        return synth.signal("c2")
    shape = (1 << c["b"],) * c["D"]
    return synth.random_signal(shape, c["seed"], c["kind"])


def _worker(rank, world, port, name):
    os.environ.setdefault("OMP_NUM_THREADS", "2")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        c = CASES[name]
        D, b, layout = c["D"], c["b"], c["layout"]
        shp = Q.shape(D, [b, b], layout)
        d = D * b
        l = int(np.log2(world))
        dl = d - l
        x = _global(c)
        part = np.ascontiguousarray(SH.shard_of(x, shp, world, rank))
        (_, _), bits = Q.qtt_shard_geometry(shp, world, rank)
        v_loc = _local_qtt(part, D, bits, layout)
        v = O.to_qtt(x, layout)
        np.testing.assert_array_equal(v_loc, v[rank << dl:(rank + 1) << dl])
        cores = sharded_tt_svd(v_loc, d, dl, c["eps"], 10, 1e-10)
        ref = O.tt_svd(v, c["eps"], 10, 1e-10)
        assert O.ranks_of(cores) == O.ranks_of(ref), (O.ranks_of(cores), O.ranks_of(ref))
        full_ref = O.full(ref)
        rel = np.linalg.norm(O.full(cores) - full_ref) / np.linalg.norm(full_ref)
        assert rel <= 1e-9, rel
        # every rank holds bitwise the same cores (the redundant steps agree)
        flat = np.concatenate([cc.reshape(-1) for cc in cores])
        g = _allgather_cols(flat.reshape(1, -1))
        np.testing.assert_array_equal(g[:, :flat.size], g[:, flat.size:])
        # sharded expansion = this rank's slice of the global expansion
        mine = O.full(fold_tail(cores, l, rank))
        np.testing.assert_allclose(mine, O.full(cores)[rank << dl:(rank + 1) << dl],
                                   rtol=0, atol=1e-13 * np.abs(full_ref).max())
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module", autouse=True)
def _lib():
    B.build()
    Q.lib()


@pytest.mark.parametrize("name", sorted(CASES))
def test_sharded_tt_svd_world2(name):
    mp.spawn(_worker, args=(2, _port(), name), nprocs=2, join=True)
