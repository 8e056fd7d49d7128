"""GPU parity of bilinear_resample with pole extension (resample.hpp:20-114) against the
reference's outputs (tests/golden) and the properties test_resample.cpp pins."""
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

DEV = torch.device("cuda", 0)
EQ, GA = 0, 1
TOL = 2e-6  # fp32 samples, fp64-derived weights


def grid(kind, nlat, nlon, last_pi=False):
    g = S.build_equiangular(nlat, nlon) if kind == EQ else S.build_gaussian(nlat, nlon)
    if last_pi:  # synthetic pole-to-pole grid (test_resample.cpp:46-47)
        col = np.array(g.colatitudes, dtype=np.float64)
        col[-1] = math.pi
        g = S.GridSpec(g.kind, g.nlat, g.nlon, col, np.array(g.longitudes), np.array(g.quad_weights))
    return g


def resample(x, gi, go):
    f = S.SphericalField(gi, torch.tensor(x, dtype=torch.float32, device=DEV))
    y = S.bilinear_resample(f, go).data
    torch.cuda.synchronize()
    return y.cpu().numpy().astype(np.float64)


CASES = {
    "ga8_eq13": (GA, 8, 16, 0, EQ, 13, 20),
    "eq9_ga7": (EQ, 9, 12, 0, GA, 7, 9),
    "eq4_eq4x6": (EQ, 4, 4, 0, EQ, 4, 6),
    "ga8_id": (GA, 8, 16, 0, GA, 8, 16),
    "eq9_id": (EQ, 9, 16, 0, EQ, 9, 16),
    "p2p4": (EQ, 4, 4, 1, EQ, 5, 8),
    "eq91_ga45": (EQ, 91, 180, 0, GA, 45, 90),
    "ga45_eq91": (GA, 45, 90, 0, EQ, 91, 180),
}


@pytest.mark.parametrize("name", list(CASES))
def test_resample_golden(golden, name):
    ik, ih, iw, lp, ok, oh, ow = CASES[name]
    x = oracle.random_field((2, ih, iw), 40)
    y = resample(x, grid(ik, ih, iw, lp), grid(ok, oh, ow))
    assert rel_l2(y, golden[f"resample_{name}"]) <= TOL, name
    assert np.abs(y - golden[f"resample_{name}"]).max() <= 1e-5


def test_resample_identity_constants_range():
    """test_resample.cpp:55-63 (identity) and :110-123 (constants, input range)."""
    for g in (grid(GA, 8, 16), grid(EQ, 9, 16)):
        u = oracle.random_field((2, g.nlat, g.nlon), 40)
        assert np.abs(resample(u, g, g) - u).max() <= 1e-6
    gi, go = grid(GA, 8, 16), grid(EQ, 13, 20)
    c = np.full((1, 8, 16), -0.7)
    assert np.abs(resample(c, gi, go) + 0.7).max() <= 1e-6
    u = oracle.random_field((1, 8, 16), 44)
    v = resample(u, gi, go)
    assert v.min() >= u.min() - 1e-6 and v.max() <= u.max() + 1e-6


def test_resample_batched_cfg_size():
    """Decoder-scale shapes (Gaussian 360x720 latent -> 721x1440 equiangular), batched
    fields, against the reference on a 2-field subset."""
    gi, go = grid(GA, 360, 720), grid(EQ, 721, 1440)
    x = oracle.random_field((3, 360, 720), 7)
    y = resample(x, gi, go)
    want = oracle.ref().bilinear_resample(GA, 360, 720, EQ, 721, 1440, x[:2]) if oracle.ref_available() else None
    if want is not None:
        assert rel_l2(y[:2], want) <= TOL
    assert y.shape == (3, 721, 1440)


SCASES = {"ga8_ga12": (GA, 8, 16, GA, 12, 24), "ga12_eq9": (GA, 12, 24, EQ, 9, 16),
          "eq9_ga8": (EQ, 9, 16, GA, 8, 16), "ga45_eq91": (GA, 45, 90, EQ, 91, 180)}


@pytest.mark.parametrize("name", list(SCASES))
def test_spectral_resample_golden(golden, name):
    """resample.hpp:120-132 through the SHT kernels (fp32 / 3xTF32 tolerance)."""
    ik, ih, iw, ok, oh, ow = SCASES[name]
    x = oracle.random_field((2, ih, iw), 41)
    f = S.SphericalField(grid(ik, ih, iw), torch.tensor(x, dtype=torch.float32, device=DEV))
    y = S.spectral_resample(f, grid(ok, oh, ow)).data
    torch.cuda.synchronize()
    assert rel_l2(y.cpu().numpy().astype(np.float64), golden[f"sresample_{name}"]) <= 1e-5, name
