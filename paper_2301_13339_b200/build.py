"""Build libqtt.so (hand-written sm_100a CUDA + the C ABI of include/qtt.h)
in-tree with nvcc.  Used by __graft_entry__.build() and the tests.

Every csrc/*.cu is compiled to an object file in parallel (the kernels of a
file call only inline device helpers, so no relocatable device code is
needed), then the objects are linked into libqtt.so."""

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libqtt.so")
OBJ = os.path.join(HERE, "build_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                 "-diag-suppress", "177"]
LDFLAGS = ARCH + ["-shared", "-ldl"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.h"))) + \
        sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + \
        [os.path.join(ROOT, "include", "qtt.h")]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def _compile(src, extra, verbose):
    obj = os.path.join(OBJ + ("_diag" if extra else ""), os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC] + CFLAGS + list(extra) + ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)
    return obj


def build(force=False, verbose=False, out=None, extra=()):
    """Compile and link.  `out` / `extra`: a diagnostic variant (e.g.
    extra=["-DQTT_XF_TIMING"]) written to another path, never the product
    library."""
    target = out or LIB
    if out is None and not extra and not force and up_to_date():
        return LIB
    os.makedirs(OBJ + ("_diag" if extra else ""), exist_ok=True)
    srcs = sources()
    with ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 4))) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra, verbose), srcs))
    cmd = [NVCC] + LDFLAGS + ["-o", target] + objs
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)
    return target


if __name__ == "__main__":
    build(force=True, verbose=True)
