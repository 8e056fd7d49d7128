"""SHT parity over field counts that select different device code paths:
  F = 1, 3 (single-CTA Legendre GEMM, odd 2F -> 16-byte quad map, EOi tile padding),
  F = 65, 130 (cta_group::2 CTA-pair GEMM, odd and even field tiles), and F = 0.
Against the fp64 C oracle (the reference's algorithm, pinned by tests/test_oracle.py) on
the cfg1 equiangular grid (forward through the dist_sht_forward 1x1 path, as the
reference) and a Gaussian grid; per-field relative L2 <= 1e-5."""
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
TOL = 1e-5
GRIDS = {"eq91": (0, 91, 180, 91, 90), "ga48": (1, 48, 96, 48, 48)}


@pytest.mark.parametrize("F", [1, 3, 65, 130])
@pytest.mark.parametrize("gname", list(GRIDS))
def test_forward_inverse_by_field_count(gname, F):
    kind, nlat, nlon, lmax, mmax = GRIDS[gname]
    g = S.build_equiangular(nlat, nlon) if kind == 0 else S.build_gaussian(nlat, nlon)
    p = S.ShtPlan(g, lmax, mmax, "3xtf32", allow_equiangular_forward=True)
    x = oracle.random_field((F, nlat, nlon), 100 + F)
    c = p.forward(torch.tensor(x, dtype=torch.float32, device=DEV), L.SPH_LAYOUT_DENSE_LM)
    y = p.inverse(c, F, L.SPH_LAYOUT_DENSE_LM)
    torch.cuda.synchronize()
    c = c.cpu().numpy().astype(np.float64)
    c = c[..., 0] + 1j * c[..., 1]
    y = y.cpu().numpy().astype(np.float64)
    o = oracle.orc()
    check = sorted({0, F // 2, F - 1})  # per-field oracle on a subset (the loop is per field)
    for f in check:
        want = o.sht_forward(kind, nlat, nlon, lmax, mmax, x[f:f + 1])
        assert rel_l2(c[f:f + 1], want) <= TOL, (gname, F, f)
        want_y = o.sht_inverse(kind, nlat, nlon, want)
        assert rel_l2(y[f:f + 1], want_y) <= TOL, (gname, F, f)


def test_zero_fields_is_a_no_op():
    g = S.build_gaussian(48, 96)
    p = S.ShtPlan(g, 48, 48, "3xtf32")
    c = p.forward(torch.zeros((0, 48, 96), device=DEV), L.SPH_LAYOUT_DENSE_LM)
    y = p.inverse(c, 0, L.SPH_LAYOUT_DENSE_LM)
    torch.cuda.synchronize()
    assert c.numel() == 0 and y.numel() == 0


def test_pair_gemm_matches_simt_anchor():
    """3xTF32 CTA-pair tcgen05 path vs the fp32 SIMT anchor at a pair-mode size."""
    g = S.build_equiangular(181, 360)
    x = torch.tensor(oracle.random_field((130, 181, 360), 7), dtype=torch.float32, device=DEV)
    outs = []
    for prec in ("3xtf32", "fp32"):
        p = S.ShtPlan(g, 181, 180, prec, allow_equiangular_forward=True)
        c = p.forward(x, L.SPH_LAYOUT_DENSE_LM)
        outs.append((c.cpu().numpy().astype(np.float64), p.inverse(c, 130, L.SPH_LAYOUT_DENSE_LM).cpu().numpy()))
    assert rel_l2(outs[0][0], outs[1][0]) <= TOL
    assert rel_l2(outs[0][1], outs[1][1]) <= TOL
    # fields at both ends of the pair tiles against the fp64 oracle
    sub = [0, 129]
    xs = x[sub].cpu().numpy().astype(np.float64)
    ref = oracle.orc().sht_forward(0, 181, 360, 181, 180, xs)
    got = outs[0][0][sub]
    assert rel_l2(got[..., 0] + 1j * got[..., 1], ref) <= TOL
    assert rel_l2(outs[0][1][sub], oracle.orc().sht_inverse(0, 181, 360, ref)) <= TOL
