"""qtt_conv_full captured in a CUDA graph (include/qtt.h "Conventions"): the
descriptor uploads are kernels, the g-chain side stream forks and joins
inside the capture, so a replay reproduces the eager result bitwise (same
kernels, same inputs, fixed reduction orders) and the replay is reusable."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2301_13339_b200 import qtt as Q  # noqa: E402
from paper_2301_13339_b200 import synth  # noqa: E402


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_conv_full_graph_replay_matches_eager(cfg):
    p = synth.problem(cfg)
    f = synth.signal(cfg)
    g = synth.kernel(p["D"], p["b"], synth.CONFIGS[cfg]["w"])
    eps = p["eps"][0]
    shp = Q.shape(p["D"], [p["b"], p["b"] if p["D"] == 2 else 0], p["layout"])
    D, F = Q.trunc(eps, p["rmax"], p["cluster_tol"]), Q.trunc(eps, p["rhat"], p["cluster_tol"])
    nb = Q.qtt_workspace_bytes(shp, D, F)
    dev = torch.device("cuda", 0)
    ws = torch.empty(nb + 256, dtype=torch.uint8, device=dev)
    fd = torch.from_numpy(np.ascontiguousarray(f).reshape(-1)).to(dev)
    gd = torch.from_numpy(np.ascontiguousarray(g).reshape(-1)).to(dev)
    y_eager = torch.empty_like(fd)
    y_graph = torch.empty_like(fd)
    s = torch.cuda.Stream(dev)

    def call(out):
        Q.qtt_conv_full(fd.data_ptr(), gd.data_ptr(), out.data_ptr(), shp, D, F, p["shift"], p["scale"],
                        ws.data_ptr(), nb, torch.cuda.current_stream(dev).cuda_stream)

    with torch.cuda.stream(s):
        call(y_eager)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        call(y_graph)
    for _ in range(2):
        y_graph.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(y_eager, y_graph)
