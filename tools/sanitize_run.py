"""Small cases that launch every kernel family of libqtt once, for
compute-sanitizer (one tool per gpurun call):

    compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_run.py
    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py
    compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py
    compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_run.py

Each case also checks the library's status word (no error bits).  GPU only;
no oracle (correctness is the parity suite's job, this run only looks for
memory errors, shared-memory races and barrier misuse under the tools).
Kernels launched: k_finish (d <= 12 and the d > 12 tail), k_level_gram,
k_level_solve, k_project<1/0>, k_gram_reduce, k_step_solve, k_transform<10>
and <16>, k_hadamard_round (in-CTA and multi-CTA right-Gram chain),
hround_big kernels, k_expand_small / k_expand_prep / k_expand_main, the
TT-RSVD sketches, the drop-off rule, the sharded kernels (k_fold_tail,
k_gather_w) through a virtual communicator, and the eigensolver test entry.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from paper_2301_13339_b200 import qtt as Q  # noqa: E402
from paper_2301_13339_b200 import shard as SH  # noqa: E402
from paper_2301_13339_b200 import synth  # noqa: E402
from gpu_util import dev, gpu_conv_full, gpu_decompose, gpu_decompose_policy, gpu_full, shape_of, stream, ws  # noqa: E402


def check(rep, what):
    bits = rep["status_bits"] if isinstance(rep, dict) else 0
    assert bits & 3 == 0, (what, bits)
    print(f"ok {what}", flush=True)


def main():
    Q.lib()
    # C1 (d = 12): whole TT-SVD in k_finish, k_transform<10>, in-CTA rounding chain, small expansion
    p = synth.problem("c1")
    f, g = synth.signal("c1"), synth.kernel(1, 12, 40.0)
    _, rep = gpu_conv_full(f, g, "1d", (1e-3, 10, 1e-10), (1e-3, 8, 1e-10), p["shift"], p["scale"])
    check(rep, "c1 conv")
    # C2 (d = 18): level Gram, level solve, projections, step solves, finish,
    # multi-CTA rounding Gram chain, k_expand_main
    p = synth.problem("c2")
    f, g = synth.signal("c2"), synth.kernel(2, 9, 60.0)
    _, rep = gpu_conv_full(f, g, "interleaved", (1e-3, 10, 1e-10), (1e-3, 8, 1e-10), p["shift"], p["scale"])
    check(rep, "c2 conv")
    # several chunks per CTA (1D / concat loaders), expansion in both layouts
    for x, lay in ((synth.random_signal((1 << 22,), 8, "smooth"), "1d"),
                   (synth.random_signal((2048, 2048), 9, "smooth"), "concat")):
        tt = gpu_decompose(x, lay, 1e-3, 10)
        gpu_full(tt, x)
        print(f"ok decompose+expand {lay} d=22", flush=True)
    # batch of 4 with a shared kernel (in-CTA rounding chain, batched decomposition)
    fb = np.stack([synth.random_signal((128, 128), 30 + i) for i in range(4)])
    gk = synth.kernel(2, 7, 30.0)
    _, rep = gpu_conv_full(fb, gk, "interleaved", (1e-3, 10, 1e-10), (1e-3, 8, 1e-10), (64, 64), 1e-4, batch=4)
    check(rep, "batch conv")
    # paper caps (10, 15): k_transform<16>, hround_big
    f1, g1 = synth.random_signal((1 << 14,), 91, "smooth"), synth.random_signal((1 << 14,), 93, "smooth")
    _, rep = gpu_conv_full(f1, g1, "1d", (1e-5, 10, 1e-10), (1e-5, 15, 1e-10), (1 << 13,), 0.25)
    check(rep, "caps (10,15) conv")
    # TT-RSVD and the drop-off rule
    x = synth.random_signal((1 << 18,), 4, "smooth")
    gpu_full(gpu_decompose_policy(x, "1d", (1e-4, 10, 1e-10, None, (5, 7))), x)
    print("ok rsvd", flush=True)
    gpu_full(gpu_decompose_policy(x, "1d", (1e-4, 10, 1e-10, 1e-3)), x)
    print("ok dropoff", flush=True)
    # sharded kernels through a virtual communicator (P = 4)
    P = 4
    f, g = synth.signal("c2"), synth.kernel(2, 9, 60.0)
    shp = shape_of(f, "interleaved")
    stack = lambda a: np.concatenate([np.ascontiguousarray(q).reshape(-1) for q in SH.split(a, shp, P)])  # noqa: E731
    comm = Q.qtt_comm_init_virtual(P)
    D, F = Q.trunc(1e-3, 10, 1e-10), Q.trunc(1e-3, 8, 1e-10)
    nb = Q.qtt_comm_workspace_bytes(shp, D, F, comm)
    w = ws(nb)
    fd, gd = dev(stack(f)), dev(stack(g))
    y = torch.empty_like(fd)
    p = synth.problem("c2")
    rep = Q.qtt_conv_full(fd.data_ptr(), gd.data_ptr(), y.data_ptr(), shp, D, F, p["shift"], p["scale"],
                          w.data_ptr(), nb, stream(), report=True, comm=comm)
    torch.cuda.synchronize()
    comm.close()
    check(rep, "virtual sharded conv P=4")
    # eigensolver test entry (width 16 and 32)
    for n in (12, 16, 20, 28):
        rng = np.random.default_rng(n)
        X = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        A = X @ X.conj().T
        a = torch.from_numpy(np.ascontiguousarray(A.T).view(np.float64).copy()).cuda()
        lam = torch.empty(n, dtype=torch.float64, device="cuda")
        U = torch.empty(2 * n * n, dtype=torch.float64, device="cuda")
        sw = torch.zeros(16, dtype=torch.int32, device="cuda")
        Q.qtt_debug_eigh(a.data_ptr(), n, lam.data_ptr(), U.data_ptr(), sw.data_ptr(), stream(), mode=2 + 8, reps=1)
        torch.cuda.synchronize()
        print(f"ok eigh n={n}", flush=True)
    print("sanitize_run done")


if __name__ == "__main__":
    main()
