"""The library's calls are stream-ordered and capture into CUDA graphs: a cfg1 SHT round
trip (the latency-bound BASELINE config) and a DISCO apply captured with
torch.cuda.CUDAGraph replay bit-identically to the eager calls -- the launch-bound small
configurations run as one graph launch instead of a tracing compiler."""
import math

import numpy as np
import pytest

from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2507_12144_b200 as S  # noqa: E402
from paper_2507_12144_b200 import _lib as L  # noqa: E402

DEV = torch.device("cuda", 0)


def test_sht_roundtrip_and_disco_capture_into_cuda_graph():
    torch.cuda.set_device(DEV)
    p = S.ShtPlan(S.build_equiangular(91, 180), 91, 90, "3xtf32", allow_equiangular_forward=True)
    F = 32
    x = torch.tensor(oracle.random_field((F, 91, 180), 1), dtype=torch.float32, device=DEV)
    c = torch.zeros(p.coeffs_elems(F, L.SPH_LAYOUT_INTERNAL), device=DEV)
    y = torch.empty_like(x)
    ws = p.workspace(F)
    op = S.DiscoOperator(S.build_equiangular(91, 180), S.build_gaussian(45, 90), S.morlet_basis(3 * math.pi / 45))
    mix = torch.tensor(oracle.random_field((8, 4, 9), 2), dtype=torch.float32, device=DEV)
    u = torch.tensor(oracle.random_field((2, 4, 91, 180), 3), dtype=torch.float32, device=DEV)
    yd = torch.empty((2, 8, 45, 90), device=DEV)
    wd = op.workspace(2, 4, 8)

    def step():
        p.forward(x, L.SPH_LAYOUT_INTERNAL, out=c, ws=ws)
        p.inverse(c, F, L.SPH_LAYOUT_INTERNAL, out=y, ws=ws)
        op.apply(u, mix, out=yd, ws=wd)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):  # warm-up: lazily built tile lists / tensor maps are host-side
            step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    y_eager, yd_eager = y.clone(), yd.clone()
    g = torch.cuda.CUDAGraph()
    launches0 = L.launch_count()
    with torch.cuda.graph(g):
        step()
    assert L.launch_count() > launches0  # the library's kernels were captured
    y.zero_()
    yd.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, y_eager)
    assert torch.equal(yd, yd_eager)
    # and the replayed results against the fp64 oracle (fields / batch items at both ends)
    xs = x.cpu().numpy().astype(np.float64)[[0, F - 1]]
    ref = oracle.orc().sht_inverse(0, 91, 180, oracle.orc().sht_forward(0, 91, 180, 91, 90, xs))
    assert rel_l2(y.cpu().numpy().astype(np.float64)[[0, F - 1]], ref) <= 1e-5
    oop = oracle.orc().disco_assemble(0, 91, 180, 1, 45, 90, 3 * math.pi / 45)
    dref = oracle.orc().disco_apply(oop, u[1].cpu().numpy().astype(np.float64), mix.cpu().numpy().astype(np.float64))
    assert rel_l2(yd[1].cpu().numpy().astype(np.float64), dref) <= 1e-5
