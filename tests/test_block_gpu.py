"""GPU parity of spectral_conv (convolution.hpp:286-304) and the neural-operator block
(model.hpp:337-370) against reference golden vectors and the CPU oracle."""
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

TOL = 1e-5
DEV = torch.device("cuda", 0)
PI = math.pi


def T(a):
    return torch.tensor(np.asarray(a), dtype=torch.float32, device=DEV)


def N(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.float64)


def test_spectral_conv_golden(golden):
    g = S.build_gaussian(16, 32)
    x = oracle.random_field((3, 16, 32), 55)
    k = oracle.random_field((2, 3, 12), 56)
    y = S.spectral_conv(S.SphericalField(g, T(x)), T(k))
    assert rel_l2(N(y.data), golden["sconv_ga16_y"]) <= TOL


def test_spectral_conv_identity_and_delta():
    """test_convolution.cpp:263-292."""
    g = S.build_gaussian(16, 32)
    rng = np.random.default_rng(33)
    c = rng.uniform(-1, 1, (1, 8, 8)) + 1j * rng.uniform(-1, 1, (1, 8, 8))
    c[:, :, 0] = c[:, :, 0].real
    c *= np.tril(np.ones((8, 8)))
    u = oracle.orc().sht_inverse(1, 16, 32, c)
    y = S.spectral_conv(S.SphericalField(g, T(u)), T(np.ones((1, 1, 16))))
    assert np.abs(N(y.data) - u).max() <= 1e-5
    with pytest.raises(ValueError):
        S.spectral_conv(S.SphericalField(S.build_equiangular(16, 32), T(u)), T(np.ones((1, 1, 16))))


def test_spectral_conv_vs_oracle_batched():
    """B = 2 samples, 24 -> 16 channels on the 45x90 Gaussian grid."""
    g = S.build_gaussian(45, 90)
    x = oracle.random_field((2, 24, 45, 90), 3)
    k = oracle.random_field((16, 24, 45), 4) / 24
    y = N(S.spectral_conv(S.SphericalField(g, T(x)), T(k)).data)
    for b in range(2):
        ref = oracle.orc().spectral_conv(1, 45, 90, k, x[b])
        assert rel_l2(y[b], ref) <= TOL


def _block_weights(glob, C=16, Cc=8, H=32):
    r = oracle.ref() if oracle.ref_available() else None
    rnd = (lambda shape, seed: r.random_uniform(shape, seed)) if r else oracle.random_field
    return dict(
        x=rnd((C, 16, 32), 90), cond=rnd((Cc, 16, 32), 91),
        convw=rnd((C, C + Cc, 16 if glob else 9), 92) * 0.2,
        w1=rnd((H, C), 93) * 0.3, b1=rnd((H,), 94) * 0.1, w2=rnd((C, H), 95) * 0.3,
        b2=rnd((C,), 96) * 0.1, sc=rnd((C,), 97))


@pytest.mark.parametrize("glob", [0, 1])
def test_block_apply_golden(golden, glob):
    w = _block_weights(glob)
    g = S.build_gaussian(16, 32)
    bw = S.BlockWeights(bool(glob), T(w["convw"]), T(w["w1"]), T(w["b1"]), T(w["w2"]), T(w["b2"]),
                        T(w["sc"]))
    op = None if glob else S.assemble_disco(g, g, S.morlet_basis(3 * PI / 16))
    y = S.block_apply(S.SphericalField(g, T(w["x"])), S.SphericalField(g, T(w["cond"])), bw, op)
    assert rel_l2(N(y.data), golden[f"block_g{glob}_y"]) <= TOL


def test_block_epilogue_vs_oracle_cfg4_width():
    """The fused MLP epilogue at the cfg4 channel widths (C = 256, H = 512) on a
    36 x 72 patch of points, against the fp64 oracle."""
    C, H, P = 256, 512, 36 * 72
    rng = np.random.default_rng(4)
    conv = rng.uniform(-1, 1, (C, 36, 72))
    x = rng.uniform(-1, 1, (C, 36, 72))
    w1 = rng.uniform(-1, 1, (H, C)) / 16
    b1 = rng.uniform(-1, 1, H) * 0.1
    w2 = rng.uniform(-1, 1, (C, H)) / 22
    b2 = rng.uniform(-1, 1, C) * 0.1
    sc = rng.uniform(-1, 1, C)
    bw = S.BlockWeights(False, None, T(w1), T(b1), T(w2), T(b2), T(sc))
    y = N(S.block_epilogue(T(conv), T(x), bw))
    ref = oracle.orc().block_epilogue(conv.reshape(C, P), x.reshape(C, P), w1, b1, w2, b2, sc)
    assert rel_l2(y.reshape(C, P) - x.reshape(C, P), ref - x.reshape(C, P)) <= TOL


def test_spectral_mix_alone_vs_numpy():
    """sph_spectral_mix: the per-degree channel mix of spectral_conv (convolution.hpp:295-302)
    on reference-layout coefficients, against the same contraction in fp64 numpy; any grid
    kind (coefficients of an equiangular field), batch 2, c_in 5 -> c_out 3."""
    rng = np.random.default_rng(7)
    lmax = mmax = 16
    B, cin, cout = 2, 5, 3
    c = rng.uniform(-1, 1, (B, cin, lmax, mmax)) + 1j * rng.uniform(-1, 1, (B, cin, lmax, mmax))
    c[..., 0] = c[..., 0].real
    c *= np.tril(np.ones((lmax, mmax)))  # zeros above the diagonal (m > l), the reference layout
    k = rng.uniform(-1, 1, (cout, cin, 20))
    out = S.spectral_mix(S.SpectralCoeffs(lmax, mmax, torch.tensor(c, dtype=torch.complex64, device=DEV)),
                         T(k), grid=S.build_equiangular(17, 32)).coeffs
    ref = np.einsum("bilm,oil->bolm", c, k[:, :, :lmax])
    got = out.cpu().numpy().astype(np.complex128)
    assert rel_l2(got, ref) <= TOL
    assert np.all(got[..., np.triu_indices(lmax, 1, mmax)[0], np.triu_indices(lmax, 1, mmax)[1]] == 0)
