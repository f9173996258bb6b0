"""Host-side plumbing of the column-sharded path (include/qtt.h "Multi-GPU",
SURVEY §8(e)): cut a global array into the shards the library expects and
put sharded outputs back together.  Pure memory movement (slicing and
concatenation); the shard placement itself comes from the library's
qtt_shard_geometry, so the C ABI stays the single authority on it.

Works on numpy arrays and torch tensors alike (basic slicing only).
"""

from . import qtt as Q


def geometry(shp, nshards):
    """[(origin (x0, y0), bits (bx, by))] for every shard."""
    return [Q.qtt_shard_geometry(shp, nshards, s) for s in range(nshards)]


def shard_of(x, shp, nshards, s):
    """Shard s of the global array x (1D: (n,), 2D: (ny, nx) row-major),
    as a view / slice with the shard's own shape."""
    (x0, y0), (bx, by) = Q.qtt_shard_geometry(shp, nshards, s)
    if shp.D == 1:
        return x[x0:x0 + (1 << bx)]
    return x[y0:y0 + (1 << by), x0:x0 + (1 << bx)]


def split(x, shp, nshards):
    """All shards of x, in shard order (each contiguous-able)."""
    return [shard_of(x, shp, nshards, s) for s in range(nshards)]


def assemble(parts, shp, nshards, out):
    """Write shard arrays `parts` (in shard order, each shaped like the
    shard) back into the global array `out`; returns out."""
    for s, p in enumerate(parts):
        (x0, y0), (bx, by) = Q.qtt_shard_geometry(shp, nshards, s)
        if shp.D == 1:
            out[x0:x0 + (1 << bx)] = p.reshape(-1)
        else:
            out[y0:y0 + (1 << by), x0:x0 + (1 << bx)] = p.reshape(1 << by, 1 << bx)
    return out
