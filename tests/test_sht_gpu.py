"""GPU parity of the SHT against the CPU oracle / reference golden vectors.

Bar (BASELINE north_star): relative L2 <= 1e-5 for the fp32 paths (3xTF32 tensor-core
and fp32 SIMT); the reduced-precision single-pass TF32 mode is stated separately
(<= 5e-3).  Test cases follow proj/tests/test_harmonics.cpp and acceptance.cpp.
"""
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

TOL = 1e-5
TOL_TF32 = 5e-3
DEV = torch.device("cuda", 0)


def plan(kind, nlat, nlon, lmax, mmax, prec="3xtf32", eq=True):
    g = S.build_equiangular(nlat, nlon) if kind == 0 else S.build_gaussian(nlat, nlon)
    return S.ShtPlan(g, lmax, mmax, prec, allow_equiangular_forward=eq)


def fwd(p, x, layout=L.SPH_LAYOUT_DENSE_LM):
    xt = torch.tensor(x, dtype=torch.float32, device=DEV)
    out = p.forward(xt, layout)
    torch.cuda.synchronize()
    if layout == L.SPH_LAYOUT_DENSE_LM:
        o = out.cpu().numpy().astype(np.float64)
        return o[..., 0] + 1j * o[..., 1]
    return out


def inv(p, c, F):
    if isinstance(c, np.ndarray):
        c = torch.tensor(np.stack([c.real, c.imag], -1), dtype=torch.float32, device=DEV)
        y = p.inverse(c, F, L.SPH_LAYOUT_DENSE_LM)
    else:
        y = p.inverse(c, F, L.SPH_LAYOUT_INTERNAL)
    torch.cuda.synchronize()
    return y.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("prec", ["3xtf32", "fp32"])
def test_cfg1_equiangular_roundtrip_vs_reference(golden, prec):
    """cfg1: 91x180 equiangular, lmax=91, mmax=90, 32 channels (seed 1)."""
    x = oracle.random_field((32, 91, 180), 1)
    p = plan(0, 91, 180, 91, 90, prec)
    c = fwd(p, x)
    assert rel_l2(c[:4], golden["cfg1_fwd"]) <= TOL
    ref = oracle.orc().sht_forward(0, 91, 180, 91, 90, x)
    assert rel_l2(c, ref) <= TOL
    # reference-layout zeros above the diagonal
    lm = np.arange(91)[:, None] < np.arange(90)[None, :]
    assert np.all(c[:, lm] == 0)
    y = inv(p, c, 32)
    assert rel_l2(y[:4], golden["cfg1_rt"]) <= TOL
    # the equiangular round trip is NOT the identity (SURVEY finding 3): compare with
    # the oracle's own round trip, never with the input
    yref = oracle.orc().sht_inverse(0, 91, 180, ref)
    assert rel_l2(y, yref) <= TOL


def test_cfg1_tf32_reduced_precision(golden):
    x = oracle.random_field((4, 91, 180), 1)
    p = plan(0, 91, 180, 91, 90, "tf32")
    c = fwd(p, x)
    e = rel_l2(c, golden["cfg1_fwd"])
    assert e <= TOL_TF32, e


def test_internal_layout_roundtrip_matches_dense():
    x = oracle.random_field((6, 91, 180), 3)
    p = plan(0, 91, 180, 91, 90)
    ci = fwd(p, x, L.SPH_LAYOUT_INTERNAL)
    y1 = inv(p, ci, 6)
    y2 = inv(p, fwd(p, x), 6)
    assert rel_l2(y1, y2) <= 1e-6


@pytest.mark.parametrize("name,kind,nlat,nlon,lmax,mmax,seed,C", [
    ("ga32", 1, 32, 64, 32, 32, 7, 2),
    ("eq9", 0, 9, 16, 9, 8, 5, 3),
])
def test_golden_roundtrips(golden, name, kind, nlat, nlon, lmax, mmax, seed, C):
    x = oracle.random_field((C, nlat, nlon), seed)
    p = plan(kind, nlat, nlon, lmax, mmax)
    c = fwd(p, x)
    assert rel_l2(c, golden[f"{name}_fwd"]) <= TOL
    y = inv(p, c, C)
    assert rel_l2(y, golden[f"{name}_rt"]) <= TOL


def test_gaussian_roundtrip_is_identity_on_bandlimited():
    """test_harmonics.cpp:116-131 (1e-11 in fp64; fp32 bar here)."""
    rng = np.random.default_rng(7)
    c = rng.uniform(-1, 1, (2, 32, 32)) + 1j * rng.uniform(-1, 1, (2, 32, 32))
    c[:, :, 0] = c[:, :, 0].real
    c *= np.tril(np.ones((32, 32)))
    p = plan(1, 32, 64, 32, 32)
    f = inv(p, c, 2)
    r = fwd(p, f)
    assert rel_l2(r, c) <= TOL


def test_mode_truncation(golden):
    x = oracle.random_field((2, 16, 32), 31)
    p = plan(1, 16, 32, 16, 8)
    assert rel_l2(fwd(p, x), golden["ga16_m8_fwd"]) <= TOL


def test_inverse_msynth_clamp(golden):
    """nlon = 10 < 2*mmax: orders >= (nlon-1)/2+1 are dropped (harmonics.hpp:179)."""
    cf = oracle.ref().random_uniform((1, 8, 8, 2), 8) if oracle.ref_available() else None
    if cf is None:
        pytest.skip("needs the reference stream")
    c = cf[..., 0] + 1j * cf[..., 1]
    p = plan(0, 9, 10, 8, 8)
    assert rel_l2(inv(p, c, 1), golden["inv_msynth"]) <= TOL


def test_constant_field_and_Y53():
    """test_harmonics.cpp:57-79."""
    g = S.build_gaussian(8, 16)
    f = torch.ones((1, 8, 16), device=DEV)
    c = S.sht_forward(S.SphericalField(g, f), 8, 8).coeffs.cpu().numpy()
    want = np.zeros((1, 8, 8), complex)
    want[0, 0, 0] = math.sqrt(4 * math.pi)
    assert np.abs(c - want).max() <= 1e-5
    th = g.colatitudes[:, None]
    ph = g.longitudes[None, :]
    y53 = -(1 / 32) * math.sqrt(385 / math.pi) * np.sin(th) ** 3 * (9 * np.cos(th) ** 2 - 1) * np.cos(3 * ph)
    c = S.sht_forward(S.SphericalField(g, torch.tensor(y53[None], dtype=torch.float32, device=DEV)),
                      8, 8).coeffs.cpu().numpy()
    want = np.zeros((1, 8, 8), complex)
    want[0, 5, 3] = 0.5
    assert np.abs(c - want).max() <= 1e-5


def test_rotation_phase_and_linearity():
    """test_harmonics.cpp:133-161."""
    g = S.build_gaussian(8, 16)
    rng = np.random.default_rng(21)
    u = rng.uniform(-1, 1, (1, 8, 16))
    v = rng.uniform(-1, 1, (1, 8, 16))
    p = plan(1, 8, 16, 8, 8)
    cu, cv = fwd(p, u), fwd(p, v)
    cw = fwd(p, 1.7 * u - 0.4 * v)
    assert np.abs(cw - (1.7 * cu - 0.4 * cv)).max() <= 1e-5
    cr = fwd(p, np.roll(u, 3, axis=-1))
    m = np.arange(8)
    phase = np.exp(-2j * np.pi * m * 3 / 16)
    assert np.abs(cr - cu * phase[None, None, :] * (np.arange(8)[:, None] >= m[None, :])).max() <= 1e-5


def test_preconditions_raise_like_reference():
    """test_harmonics.cpp:174-181."""
    g = S.build_gaussian(8, 16)
    f = S.SphericalField(g, torch.zeros((1, 8, 16), device=DEV))
    with pytest.raises(ValueError):
        S.sht_forward(f, 9, 8)
    with pytest.raises(ValueError):
        S.sht_forward(f, 8, 9)
    e = S.build_equiangular(8, 16)
    with pytest.raises(ValueError):
        S.sht_forward(S.SphericalField(e, torch.zeros((1, 8, 16), device=DEV)), 8, 8)
    # and the raw C ABI without the equiangular flag
    p = plan(0, 8, 16, 8, 8, eq=False)
    with pytest.raises(ValueError):
        p.forward(torch.zeros((1, 8, 16), device=DEV))


def test_zero_inverse_is_zero():
    p = plan(0, 9, 16, 6, 6)
    y = inv(p, np.zeros((1, 6, 6), complex), 1)
    assert np.all(y == 0)


def test_cfg2_721_subset_and_properties():
    """721x1440 equiangular, lmax=721, mmax=720: two fields against the oracle (the
    per-field loop makes a subset exact), plus size-independent properties on a
    larger batch: linearity and INTERNAL/DENSE agreement."""
    x = oracle.random_field((2, 721, 1440), 1)
    p = plan(0, 721, 1440, 721, 720)
    c = fwd(p, x)
    ref = oracle.orc().sht_forward(0, 721, 1440, 721, 720, x)
    assert rel_l2(c, ref) <= TOL
    y = inv(p, c, 2)
    yref = oracle.orc().sht_inverse(0, 721, 1440, ref)
    assert rel_l2(y, yref) <= TOL
    # linearity at full size through the internal layout
    xt = torch.tensor(x, dtype=torch.float32, device=DEV)
    a = p.forward(xt, L.SPH_LAYOUT_INTERNAL)
    b = p.forward(2.0 * xt, L.SPH_LAYOUT_INTERNAL)
    torch.cuda.synchronize()
    assert float((b - 2 * a).norm() / (2 * a).norm()) <= 1e-6


@pytest.mark.parametrize("cluster", ["1", "2", "4"])
def test_gemm_cluster_multicast_matches_simt(monkeypatch, cluster):
    """The table-multicast cluster path of the tcgen05 GEMM (used at benchmark batch
    sizes) against the fp32 SIMT anchor on the same inputs: 512 fields of cfg1."""
    monkeypatch.setenv("SPH_GEMM_CLUSTER", cluster)
    x = oracle.random_field((512, 91, 180), 9)
    a = fwd(plan(0, 91, 180, 91, 90, "3xtf32"), x)
    b = fwd(plan(0, 91, 180, 91, 90, "fp32"), x)
    assert rel_l2(a, b) <= 2e-6
    pa = plan(0, 91, 180, 91, 90, "3xtf32")
    ya = inv(pa, a, 512)
    yb = inv(plan(0, 91, 180, 91, 90, "fp32"), a, 512)
    assert rel_l2(ya, yb) <= 2e-6
    # and both ends of the batch against the fp64 oracle (not only the SIMT anchor)
    sub = [0, 255, 511]
    ref = oracle.orc().sht_forward(0, 91, 180, 91, 90, x[sub])
    assert rel_l2(a[sub], ref) <= TOL
    assert rel_l2(ya[sub], oracle.orc().sht_inverse(0, 91, 180, a[sub])) <= TOL


# ------------------------------------------------------------- SHT adjoints
def _grid(kind, nlat, nlon):
    return S.build_gaussian(nlat, nlon) if kind == 1 else S.build_equiangular(nlat, nlon)


@pytest.mark.parametrize("kind,nlat,nlon,lmax,mmax", [(1, 12, 24, 12, 9), (0, 9, 16, 9, 8), (1, 45, 90, 45, 45)])
def test_sht_adjoints_vs_oracle(kind, nlat, nlon, lmax, mmax):
    """SPH_FLAG_ADJOINT plans against the fp64 oracle restatement of the adjoint formulas
    (tests/test_oracle.py::test_sht_adjoint_formulas pins those by the adjoint identity)."""
    dev = torch.device("cuda", 0)
    o = oracle.orc()
    colat, w = o.grid(kind, nlat, nlon)
    rng = np.random.default_rng(3)
    z = rng.standard_normal((3, nlat, nlon))
    d = (rng.standard_normal((3, lmax, mmax)) + 1j * rng.standard_normal((3, lmax, mmax))) * \
        (np.tril(np.ones((lmax, mmax))) > 0)
    g = _grid(kind, nlat, nlon)
    # S^T z
    c = S.sht_inverse_adjoint(S.SphericalField(g, torch.tensor(z, dtype=torch.float32, device=dev)), lmax, mmax)
    out = np.zeros((3, lmax, mmax, 2))
    assert o.L.orc_sht_forward(nlat, nlon, colat, np.ones(nlat), lmax, mmax, 3, np.ascontiguousarray(z), out) == 0
    ref = (out[..., 0] + 1j * out[..., 1]) * np.where(np.arange(mmax) >= 1, 2.0, 1.0)
    assert rel_l2(c.coeffs.cpu().numpy().astype(np.complex128), ref) <= TOL
    if kind == 1:  # A^T d
        y = S.sht_forward_adjoint(S.SpectralCoeffs(lmax, mmax, torch.tensor(d, dtype=torch.complex64, device=dev)), g)
        ref = w[None, :, None] * o.sht_inverse(kind, nlat, nlon, d * np.where(np.arange(mmax) >= 1, 0.5, 1.0))
        assert rel_l2(y.data.cpu().numpy().astype(np.float64), ref) <= TOL


def test_sht_adjoint_identities_latent_size():
    """<A x, d> = <x, A^T d> and <S c, z> = <c, S^T z> through the kernels at the
    360x720 Gaussian latent grid (lmax = mmax = 360), fp32 tolerance."""
    dev = torch.device("cuda", 0)
    g = S.build_gaussian(360, 720)
    gen = torch.Generator(device="cpu").manual_seed(11)
    x = torch.randn(2, 360, 720, generator=gen).to(dev)
    z = torch.randn(2, 360, 720, generator=gen).to(dev)
    tri = torch.tril(torch.ones(360, 360)).to(dev)
    d = torch.complex(torch.randn(2, 360, 360, generator=gen), torch.randn(2, 360, 360, generator=gen)).to(dev) * tri
    c = torch.complex(torch.randn(2, 360, 360, generator=gen), torch.randn(2, 360, 360, generator=gen)).to(dev) * tri
    Ax = S.sht_forward(S.SphericalField(g, x), 360, 360).coeffs
    ATd = S.sht_forward_adjoint(S.SpectralCoeffs(360, 360, d), g).data
    lhs = (Ax.conj() * d).real.double().sum().item()
    rhs = (x.double() * ATd.double()).sum().item()
    assert abs(lhs - rhs) <= 2e-5 * (Ax.abs().double().pow(2).sum().sqrt() * d.abs().double().pow(2).sum().sqrt()).item()
    Sc = S.sht_inverse(S.SpectralCoeffs(360, 360, c), g).data
    STz = S.sht_inverse_adjoint(S.SphericalField(g, z), 360, 360).coeffs
    lhs = (Sc.double() * z.double()).sum().item()
    rhs = (c.conj() * STz).real.double().sum().item()
    assert abs(lhs - rhs) <= 2e-5 * (Sc.double().pow(2).sum().sqrt() * z.double().pow(2).sum().sqrt()).item()
