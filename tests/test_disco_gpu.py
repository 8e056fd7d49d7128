"""GPU parity of DISCO (convolution.hpp:141-220) against reference golden vectors and
the CPU oracle.  Both device paths: the default longitude-Fourier path (3xTF32 channel
mix) and the fp32 direct-gather anchor.  Cases follow proj/tests/test_convolution.cpp."""
import math
import os

import numpy as np
import pytest

from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2507_12144_b200 as S  # noqa: E402

TOL = 1e-5
DEV = torch.device("cuda", 0)
PI = math.pi
EQ, GA = 0, 1


def grid(kind, nlat, nlon):
    return S.build_equiangular(nlat, nlon) if kind == EQ else S.build_gaussian(nlat, nlon)


def apply(op, x, mix):
    y = op.apply(torch.tensor(x, dtype=torch.float32, device=DEV),
                 torch.tensor(mix, dtype=torch.float32, device=DEV))
    torch.cuda.synchronize()
    return y.cpu().numpy().astype(np.float64)


CASES = {
    "ga16_ga8": (GA, 16, 32, GA, 8, 16, 3 * PI / 8, 3, 2),
    "eq16_eq16": (EQ, 16, 32, EQ, 16, 32, 4 * PI / 16, 3, 2),
    "eq12_stride3": (EQ, 12, 24, EQ, 12, 8, 3 * PI / 12, 1, 1),
    "eq91_ga45": (EQ, 91, 180, GA, 45, 90, 3 * PI / 45, 4, 8),
    "eq9_eq9": (EQ, 9, 16, EQ, 9, 16, 3 * PI / 9, 2, 1),
}


@pytest.mark.parametrize("prec", ["3xtf32", "fp32"])
@pytest.mark.parametrize("name", list(CASES))
def test_disco_golden(golden, name, prec):
    ik, ih, iw, ok, oh, ow, cut, cin, cout = CASES[name]
    op = S.DiscoOperator(grid(ik, ih, iw), grid(ok, oh, ow), S.morlet_basis(cut), prec)
    assert op.n_basis == 9
    assert op.nnz_per_basis == int(golden[f"disco_{name}_rows"].sum())
    mix = oracle.random_field((cout, cin, 9), 77)
    x = oracle.random_field((cin, ih, iw), 78)
    y = apply(op, x[None], mix)[0]
    assert rel_l2(y, golden[f"disco_{name}_y"]) <= TOL, name


def test_disco_batch_and_isotropic(golden):
    op = S.DiscoOperator(grid(EQ, 12, 24), grid(EQ, 12, 24), S.isotropic_basis(PI / 12))
    assert op.n_basis == 1
    x = oracle.random_field((1, 12, 24), 5)
    y = apply(op, np.stack([x, 2 * x]), np.ones((1, 1, 1)))
    assert rel_l2(y[0], golden["disco_iso_eq12_y"]) <= TOL
    assert rel_l2(y[1], 2 * golden["disco_iso_eq12_y"]) <= TOL


def test_disco_shift_equivariance():
    """test_convolution.cpp:187-212 (bitwise in fp64; tolerance here, stride 3)."""
    op = S.DiscoOperator(grid(EQ, 12, 24), grid(EQ, 12, 8), S.morlet_basis(3 * PI / 12))
    assert op.stride == 3
    mix = oracle.random_field((1, 1, 9), 13)
    u = oracle.random_field((1, 1, 12, 24), 14)
    y = apply(op, u, mix)
    yr = apply(op, np.roll(u, 3, axis=-1), mix)
    assert rel_l2(yr, np.roll(y, 1, axis=-1)) <= 1e-6


def test_disco_zero_input():
    op = S.DiscoOperator(grid(GA, 8, 16), grid(GA, 8, 16), S.morlet_basis(3 * PI / 8))
    y = apply(op, np.zeros((1, 2, 8, 16)), oracle.random_field((2, 2, 9), 3))
    assert np.all(y == 0)


def test_disco_rejects_like_reference():
    """test_convolution.cpp:247-261."""
    with pytest.raises(ValueError):
        S.DiscoOperator(grid(GA, 8, 16), grid(GA, 4, 8), S.isotropic_basis(1e-4))
    with pytest.raises(ValueError):
        S.DiscoOperator(grid(GA, 8, 16), grid(GA, 8, 12), S.isotropic_basis(1.0))
    with pytest.raises(ValueError):
        S.morlet_basis(0.0)


def test_disco_cfg3_structure_and_subset(golden):
    """cfg3: 721x1440 equiangular -> 360x720 Gaussian, Morlet, cutoff 3pi/360.  The
    assembled row structure equals the reference's (158,266 entries per basis
    function); a 2 -> 3 channel subset of the apply matches the oracle."""
    op = S.DiscoOperator(grid(EQ, 721, 1440), grid(GA, 360, 720), S.morlet_basis(3 * PI / 360))
    assert op.nnz_per_basis == int(golden["disco_cfg3_rows"].sum()) == 158266
    assert op.stride == 2
    x = oracle.random_field((2, 721, 1440), 1)
    mix = oracle.random_field((3, 2, 9), 77)
    y = apply(op, x[None], mix)[0]
    oop = oracle.orc().disco_assemble(EQ, 721, 1440, GA, 360, 720, 3 * PI / 360)
    ref = oracle.orc().disco_apply(oop, x, mix)
    assert rel_l2(y, ref) <= TOL


def test_disco_fourier_vs_direct_anchor_full_size():
    """Size-independent check at the benchmark shape: the Fourier path equals the
    reference-order direct gather (fp32 anchor) on 64 -> 32 channels, batch 2."""
    gi, go = grid(EQ, 721, 1440), grid(GA, 360, 720)
    a = S.DiscoOperator(gi, go, S.morlet_basis(3 * PI / 360), "3xtf32")
    b = S.DiscoOperator(gi, go, S.morlet_basis(3 * PI / 360), "fp32")
    g = torch.Generator(device=DEV).manual_seed(5)
    x = torch.rand((2, 64, 721, 1440), device=DEV, generator=g) * 2 - 1
    mix = (torch.rand((32, 64, 9), device=DEV, generator=g) * 2 - 1) / 24
    ya, yb = a.apply(x, mix), b.apply(x, mix)
    torch.cuda.synchronize()
    assert float((ya - yb).norm() / yb.norm()) <= TOL
    # output channels {0, 31} of sample 1 against the unmodified reference / fp64 oracle
    outs = [0, 31]
    xs = x[1].cpu().numpy().astype(np.float64)
    ms = mix.cpu().numpy().astype(np.float64)[outs]
    if oracle.ref_available():
        _, _, ref = oracle.ref().bench_disco(EQ, 721, 1440, GA, 360, 720, 3 * PI / 360, xs, ms,
                                             os.cpu_count() or 1, want_y=True)
    else:
        oop = oracle.orc().disco_assemble(EQ, 721, 1440, GA, 360, 720, 3 * PI / 360)
        ref = oracle.orc().disco_apply(oop, xs, ms)
    assert rel_l2(ya[1, outs].cpu().numpy().astype(np.float64), ref) <= TOL


# ------------------------------------------------ disco_transpose_apply (convolution.hpp:226-266)
def transpose(op, v, mix):
    y = op.transpose_apply(torch.tensor(v, dtype=torch.float32, device=DEV),
                           torch.tensor(mix, dtype=torch.float32, device=DEV))
    torch.cuda.synchronize()
    return y.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("prec", ["3xtf32", "fp32"])
@pytest.mark.parametrize("name", list(CASES))
def test_disco_transpose_golden(golden, name, prec):
    """Reference disco_transpose_apply outputs (tests/golden/make_golden.py)."""
    ik, ih, iw, ok, oh, ow, cut, cin, cout = CASES[name]
    op = S.DiscoOperator(grid(ik, ih, iw), grid(ok, oh, ow), S.morlet_basis(cut), prec)
    mix = oracle.random_field((cout, cin, 9), 77)
    v = oracle.random_field((cout, oh, ow), 79)
    yt = transpose(op, v[None], mix)[0]
    assert rel_l2(yt, golden[f"disco_{name}_yT"]) <= TOL, name


def _quad_dot(a, b, w):
    return float(np.einsum("chw,chw,h->", a, b, w))


@pytest.mark.parametrize("case", [
    (GA, 16, 32, GA, 8, 16, 3 * PI / 8, 2, 3),          # test_convolution.cpp:214-234
    (EQ, 91, 180, GA, 45, 90, 3 * PI / 45, 4, 8),
    (EQ, 721, 1440, GA, 360, 720, 3 * PI / 360, 4, 8),  # cfg3 grids, reduced channels
])
def test_disco_adjoint_identity(case):
    """<A u, v>_out == <u, A^T v>_in under the grids' quadrature weights."""
    ik, ih, iw, ok, oh, ow, cut, cin, cout = case
    gi, go = grid(ik, ih, iw), grid(ok, oh, ow)
    op = S.DiscoOperator(gi, go, S.morlet_basis(cut))
    mix = oracle.random_field((cout, cin, 9), 15)
    u = oracle.random_field((cin, ih, iw), 16)
    v = oracle.random_field((cout, oh, ow), 17)
    au = apply(op, u[None], mix)[0]
    bv = transpose(op, v[None], mix)[0]
    lhs = _quad_dot(au, v, np.asarray(go.quad_weights))
    rhs = _quad_dot(u, bv, np.asarray(gi.quad_weights))
    assert abs(lhs - rhs) <= 1e-5 * max(1.0, abs(lhs)), (lhs, rhs)


def test_disco_isotropic_transpose_equals_forward():
    """test_convolution.cpp:236-245 (equal Gaussian grids, isotropic basis)."""
    g = grid(GA, 10, 20)
    op = S.DiscoOperator(g, g, S.isotropic_basis(3 * PI / 10))
    mix = np.full((1, 1, 1), 0.7)
    u = oracle.random_field((1, 10, 20), 21)
    fwd = apply(op, u[None], mix)[0]
    tra = transpose(op, u[None], mix)[0]
    assert rel_l2(tra, fwd) <= TOL


def test_disco_transpose_batch_and_rejects():
    ik, ih, iw, ok, oh, ow, cut, cin, cout = CASES["ga16_ga8"]
    op = S.DiscoOperator(grid(ik, ih, iw), grid(ok, oh, ow), S.morlet_basis(cut))
    mix = oracle.random_field((cout, cin, 9), 77)
    v = oracle.random_field((cout, oh, ow), 79)
    y = transpose(op, np.stack([v, -3 * v]), mix)
    assert rel_l2(y[1], -3 * y[0]) <= TOL
    with pytest.raises(S.SphInvalidArgument):  # convolution.hpp:229-233
        op.transpose_apply(torch.zeros((1, cout + 1, oh, ow), device=DEV),
                           torch.zeros((cout, cin, 9), device=DEV))
    with pytest.raises(S.SphInvalidArgument):
        op.transpose_apply(torch.zeros((1, cout, oh, ow), device=DEV),
                           torch.zeros((cout, cin, 5), device=DEV))


@pytest.mark.parametrize("cin,cout,B", [(66, 5, 2), (130, 3, 1), (7, 4, 3), (2, 1, 1)])
def test_disco_channel_counts_vs_oracle(cin, cout, B):
    """Band kernels across channel-pass boundaries: more than 64 channels (a partial second
    64-channel pass), odd counts (the scalar kernel, channel-major U), and tiny counts;
    stride-2 grids, against the fp64 restatement."""
    op = S.DiscoOperator(grid(EQ, 12, 24), grid(GA, 6, 12), S.morlet_basis(3 * PI / 12))
    oop = oracle.orc().disco_assemble(EQ, 12, 24, GA, 6, 12, 3 * PI / 12)
    u = oracle.random_field((B, cin, 12, 24), 31)
    mix = oracle.random_field((cout, cin, 9), 32) / math.sqrt(cin)
    y = op.apply(torch.tensor(u, dtype=torch.float32, device=DEV), torch.tensor(mix, dtype=torch.float32, device=DEV))
    torch.cuda.synchronize()
    y = y.cpu().numpy().astype(np.float64)
    for b in range(B):
        ref = oracle.orc().disco_apply(oop, u[b], mix)
        assert rel_l2(y[b], ref) <= TOL, (cin, cout, b)
