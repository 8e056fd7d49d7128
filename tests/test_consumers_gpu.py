"""GPU parity of the SHT consumers against the reference's outputs:
angular_psd (metrics.hpp:300-314) and spectral_crps_loss (loss.hpp:37-81)."""
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
TOL = 1e-5


def field(x, nlat, nlon):
    return S.SphericalField(S.build_gaussian(nlat, nlon), torch.tensor(x, dtype=torch.float32, device=DEV))


@pytest.mark.parametrize("nlat,nlon,seed,key", [(16, 32, 60, "psd_ga16"), (45, 90, 61, "psd_ga45")])
def test_angular_psd_golden(golden, nlat, nlon, seed, key):
    C = 3 if nlat == 16 else 2
    x = oracle.random_field((C, nlat, nlon), seed)
    psd = S.angular_psd(field(x, nlat, nlon)).cpu().numpy().astype(np.float64)
    assert psd.shape == (C, nlat)
    assert rel_l2(psd, golden[key]) <= TOL


def test_angular_psd_rejects_equiangular():
    g = S.build_equiangular(9, 16)
    with pytest.raises(S.SphInvalidArgument):
        S.angular_psd(S.SphericalField(g, torch.zeros((1, 9, 16), device=DEV)))


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_spectral_crps_golden(golden, variant):
    ens = oracle.random_field((5, 2, 16, 32), 62)
    obs = oracle.random_field((2, 16, 32), 63)
    name = ["cdf", "spread_skill", "fair"][variant]
    got = S.spectral_crps_loss(torch.tensor(ens, dtype=torch.float32, device=DEV), field(obs, 16, 32),
                               0, name).cpu().numpy()
    assert rel_l2(got, golden[f"scrps_ga16_v{variant}"]) <= TOL


def test_spectral_crps_larger_lmax_sum(golden):
    ens = oracle.random_field((8, 3, 45, 90), 64)
    obs = oracle.random_field((3, 45, 90), 65)
    got = S.spectral_crps_loss(torch.tensor(ens, dtype=torch.float32, device=DEV), field(obs, 45, 90),
                               20, "fair").cpu().numpy()
    assert rel_l2(got, golden["scrps_ga45_v2_l20"]) <= TOL


@pytest.mark.parametrize("name,kind,nlat,nlon,lmax", [("ga24", 1, 24, 48, 24), ("eq33", 0, 33, 64, 32)])
def test_noise_field_synthesis(golden, name, kind, nlat, nlon, lmax):
    """noise.hpp:95-97: noise_field(state) = sht_inverse(state.coeffs); the GPU synthesizes
    the reference's own AR(1) noise states (3 channels) in one batched inverse SHT."""
    g = S.build_equiangular(nlat, nlon) if kind == 0 else S.build_gaussian(nlat, nlon)
    c = golden[f"noise_{name}_coeffs"]  # [C][lmax][lmax][2]
    p = S.ShtPlan(g, lmax, lmax, "3xtf32", allow_equiangular_forward=True)
    y = p.inverse(torch.tensor(c, dtype=torch.float32, device=DEV), c.shape[0])
    torch.cuda.synchronize()
    assert rel_l2(y.cpu().numpy().astype(np.float64), golden[f"noise_{name}_field"]) <= TOL
