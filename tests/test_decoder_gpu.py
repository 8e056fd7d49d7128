"""GPU parity of the fused decoder (model.hpp:372-394 decode_preclamp per channel group:
disco_apply(dec_op, bilinear_resample(latent, out_grid), mix)) against the reference's own
composition (tests/golden decoder_*), the unfused two-stage path and the fp32 precision."""
import math

import numpy as np
import pytest

from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_12144_b200 as S  # noqa: E402

DEV = torch.device("cuda", 0)
EQ, GA = 0, 1
PI = math.pi
TOL = 1e-5  # north_star fp32 tolerance (relative L2)

CASES = {
    "ga8_eq17": (GA, 8, 16, EQ, 17, 32, 3 * PI / 16, 3, 2),
    "ga6_ga12": (GA, 6, 12, GA, 12, 36, 3 * PI / 12, 2, 3),
    "eq5_eq9": (EQ, 5, 8, EQ, 9, 16, 3 * PI / 9, 2, 1),
    "eq9_eq9x24": (EQ, 9, 16, EQ, 9, 24, 3 * PI / 9, 2, 2),
    "ga45_eq91": (GA, 45, 90, EQ, 91, 180, 3 * PI / 90, 4, 1),
}


def grid(kind, nlat, nlon):
    return S.build_equiangular(nlat, nlon) if kind == EQ else S.build_gaussian(nlat, nlon)


def t(a):
    return torch.tensor(np.asarray(a), dtype=torch.float32, device=DEV)


@pytest.mark.parametrize("prec", ["3xtf32", "fp32"])
@pytest.mark.parametrize("name", list(CASES))
def test_decoder_golden(golden, name, prec):
    lk, lh, lw, ok, oh, ow, cut, cin, cout = CASES[name]
    go = grid(ok, oh, ow)
    op = S.DiscoOperator(go, go, S.morlet_basis(cut), prec)
    lat = S.SphericalField(grid(lk, lh, lw), t(golden[f"decoder_{name}_latent"]))
    y = S.decode_preclamp(op, lat, t(golden[f"decoder_{name}_mix"])).data
    torch.cuda.synchronize()
    ref = golden[f"decoder_{name}_y"]
    assert tuple(y.shape) == ref.shape
    assert rel_l2(y.cpu().numpy().astype(np.float64), ref) <= TOL, name


def test_decoder_matches_two_stage_batched_groups():
    """cfg-like shapes at reduced size: 2 batches, two channel groups with different mixes;
    the fused path equals bilinear_resample followed by disco_apply group by group."""
    gl, go = grid(GA, 45, 90), grid(EQ, 91, 180)
    op = S.DiscoOperator(go, go, S.morlet_basis(3 * PI / 90))
    g = torch.Generator(device="cpu").manual_seed(5)
    lat = torch.randn(2, 7, 45, 90, generator=g).to(DEV)
    m0 = (torch.randn(1, 4, op.n_basis, generator=g) * 0.3).to(DEV)
    m1 = (torch.randn(3, 3, op.n_basis, generator=g) * 0.3).to(DEV)
    y = S.decode_preclamp(op, S.SphericalField(gl, lat), [m0, m1]).data
    up = S.bilinear_resample(S.SphericalField(gl, lat), go).data
    y0 = op.apply(up[:, :4].contiguous(), m0)
    y1 = op.apply(up[:, 4:].contiguous(), m1)
    ref = torch.cat([y0, y1], dim=1)
    torch.cuda.synchronize()
    assert y.shape == (2, 4, 91, 180)
    err = (torch.linalg.vector_norm(y - ref) / torch.linalg.vector_norm(ref)).item()
    assert err <= 2e-6, err


def test_decoder_errors():
    go = grid(EQ, 17, 32)
    op = S.DiscoOperator(go, go, S.morlet_basis(3 * PI / 16))
    lat = S.SphericalField(grid(GA, 8, 16), torch.zeros(3, 8, 16, device=DEV))
    with pytest.raises(S.SphInvalidArgument):
        S.decode_preclamp(op, lat, torch.zeros(1, 2, op.n_basis, device=DEV))  # groups != channels
    other = S.DiscoOperator(grid(EQ, 17, 32), grid(EQ, 9, 16), S.morlet_basis(3 * PI / 9))
    with pytest.raises(S.SphInvalidArgument):
        S.DecoderPlan(other, grid(GA, 8, 16))  # not an output-grid self map


@pytest.mark.parametrize("cin", [66, 5])
def test_decoder_channel_counts(cin):
    """Fused decoder across the band kernel's 64-channel passes (66) and an odd count (the
    channel-major spectrum): equal to bilinear_resample followed by disco_apply."""
    gl, go = grid(GA, 8, 16), grid(EQ, 17, 32)
    op = S.DiscoOperator(go, go, S.morlet_basis(3 * PI / 16))
    g = torch.Generator(device="cpu").manual_seed(9)
    lat = torch.randn(2, cin, 8, 16, generator=g).to(DEV)
    mix = (torch.randn(3, cin, op.n_basis, generator=g) / math.sqrt(cin)).to(DEV)
    y = S.decode_preclamp(op, S.SphericalField(gl, lat), mix).data
    ref = op.apply(S.bilinear_resample(S.SphericalField(gl, lat), go).data, mix)
    torch.cuda.synchronize()
    err = (torch.linalg.vector_norm(y - ref) / torch.linalg.vector_norm(ref)).item()
    assert err <= 2e-6, err
