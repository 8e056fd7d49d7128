"""Out-of-bounds write checks without compute-sanitizer (closed on this GPU pool).

Every output and workspace buffer of the hot-path entry points is carved from the middle
of a larger allocation whose margins hold a sentinel; after the call (and a device
synchronize) the margins must be untouched and the results must still match the fp64
oracle.  Shapes are odd on purpose (field / channel counts, lmax not a multiple of the
32-wide tiles, partial M tiles) so that every tile-edge predicate is exercised.
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

DEV = torch.device("cuda", 0)
PAD = 1 << 16  # guard elements on each side (covers a whole 64 KB TMA box overrun)
F32_SENT = 1.2345e30
U8_SENT = 0xA5
PI = math.pi


class Guarded:
    """n elements of dtype in the middle of a sentinel-filled allocation."""

    def __init__(self, n, dtype=torch.float32, shape=None, zero=False):
        sent = F32_SENT if dtype == torch.float32 else U8_SENT
        self.buf = torch.full((n + 2 * PAD,), sent, dtype=dtype, device=DEV)
        self.sent = sent
        self.n = n
        self.view = self.buf[PAD:PAD + n]
        if zero:
            self.view.zero_()
        if shape is not None:
            self.view = self.view.view(shape)

    def intact(self):
        torch.cuda.synchronize()
        lo = bool((self.buf[:PAD] == self.sent).all())
        hi = bool((self.buf[PAD + self.n:] == self.sent).all())
        return lo and hi


def _grid(kind, nlat, nlon):
    return S.build_equiangular(nlat, nlon) if kind == 0 else S.build_gaussian(nlat, nlon)


@pytest.mark.parametrize("kind,nlat,nlon,lmax,mmax,F", [
    (0, 91, 180, 91, 90, 5),       # cfg1 grid, odd field count
    (1, 45, 90, 45, 45, 3),        # Gaussian, lmax not a multiple of 32
    (0, 181, 360, 181, 180, 131),  # pair-mode M tiles with a partial last tile
    (0, 721, 1440, 721, 720, 3),   # benchmark grid
])
def test_sht_writes_stay_in_bounds(kind, nlat, nlon, lmax, mmax, F):
    p = S.ShtPlan(_grid(kind, nlat, nlon), lmax, mmax, "3xtf32", allow_equiangular_forward=True)
    x = oracle.random_field((F, nlat, nlon), 17 + F)
    xt = torch.tensor(x, dtype=torch.float32, device=DEV)
    nws = p.workspace(F).numel()
    for layout in (L.SPH_LAYOUT_DENSE_LM, L.SPH_LAYOUT_INTERNAL):
        ne = p.coeffs_elems(F, layout)
        c = Guarded(ne, zero=True)
        ws = Guarded(nws, torch.uint8)
        p.forward(xt, layout, out=c.view, ws=ws.view)
        assert c.intact() and ws.intact(), ("forward", layout)
        y = Guarded(F * nlat * nlon, shape=(F, nlat, nlon))
        ws2 = Guarded(nws, torch.uint8)
        p.inverse(c.view, F, layout, out=y.view, ws=ws2.view)
        assert y.intact() and ws2.intact(), ("inverse", layout)
        if layout == L.SPH_LAYOUT_DENSE_LM:
            sub = [0, F - 1]
            ref = oracle.orc().sht_forward(kind, nlat, nlon, lmax, mmax, x[sub])
            got = c.view.view(F, lmax, mmax, 2).cpu().numpy().astype(np.float64)[sub]
            assert rel_l2(got[..., 0] + 1j * got[..., 1], ref) <= 1e-5
            yref = oracle.orc().sht_inverse(kind, nlat, nlon, ref)
            assert rel_l2(y.view.cpu().numpy().astype(np.float64)[sub], yref) <= 1e-5


@pytest.mark.parametrize("ik,ih,iw,ok,oh,ow,cin,cout,B", [
    (0, 91, 180, 1, 45, 90, 3, 5, 2),   # odd channel counts (scalar band kernel)
    (0, 91, 180, 1, 45, 90, 4, 6, 3),   # even channels (pair kernels)
    (1, 32, 64, 1, 32, 64, 2, 3, 1),    # equal grids
])
def test_disco_writes_stay_in_bounds(ik, ih, iw, ok, oh, ow, cin, cout, B):
    op = S.DiscoOperator(_grid(ik, ih, iw), _grid(ok, oh, ow), S.morlet_basis(3 * PI / oh))
    x = oracle.random_field((B, cin, ih, iw), 23)
    mix = oracle.random_field((cout, cin, 9), 24)
    xt = torch.tensor(x, dtype=torch.float32, device=DEV)
    mt = torch.tensor(mix, dtype=torch.float32, device=DEV)
    y = Guarded(B * cout * oh * ow, shape=(B, cout, oh, ow))
    ws = Guarded(op.workspace(B, cin, cout).numel(), torch.uint8)
    op.apply(xt, mt, out=y.view, ws=ws.view)
    assert y.intact() and ws.intact()
    oop = oracle.orc().disco_assemble(ik, ih, iw, ok, oh, ow, 3 * PI / oh)
    ref = oracle.orc().disco_apply(oop, x[B - 1], mix)
    assert rel_l2(y.view[B - 1].cpu().numpy().astype(np.float64), ref) <= 1e-5
    # adjoint
    v = torch.tensor(oracle.random_field((B, cout, oh, ow), 25), dtype=torch.float32, device=DEV)
    u = Guarded(B * cin * ih * iw, shape=(B, cin, ih, iw))
    nt = int(L.lib.sph_disco_transpose_workspace_bytes(op.h, B, cin, cout))
    wst = Guarded(max(nt, 1), torch.uint8)
    op.transpose_apply(v, mt, out=u.view, ws=wst.view)
    assert u.intact() and wst.intact()
    vref = oracle.orc().disco_transpose_apply(oop, v[B - 1].cpu().numpy().astype(np.float64), mix)
    assert rel_l2(u.view[B - 1].cpu().numpy().astype(np.float64), vref) <= 1e-5


def test_resample_and_decoder_writes_stay_in_bounds():
    """bilinear_resample and the fused decoder group (360x720 latent -> 721x1440, odd channel
    counts): guards intact and the guarded results equal to the plain calls (parity against
    the reference composition is pinned in test_resample_gpu.py / test_decoder_gpu.py)."""
    gl, go = S.build_gaussian(45, 90), S.build_equiangular(91, 180)
    B, cin, cout = 2, 3, 5
    lat = torch.tensor(oracle.random_field((B, cin, 45, 90), 31), dtype=torch.float32, device=DEV)
    rp = S.ResamplePlan(gl, go)
    r = Guarded(B * cin * 91 * 180, shape=(B, cin, 91, 180))
    rp.apply(lat, out=r.view)
    assert r.intact()
    assert torch.equal(r.view, rp.apply(lat))
    op = S.DiscoOperator(go, go, S.morlet_basis(3 * PI / 90))
    dp = S.DecoderPlan(op, gl)
    mix = torch.tensor(oracle.random_field((cout, cin, 9), 32), dtype=torch.float32, device=DEV)
    y = Guarded(B * cout * 91 * 180, shape=(B, cout, 91, 180))
    ws = Guarded(int(L.lib.sph_decoder_workspace_bytes(dp.h, B, cin, cout)), torch.uint8)
    dp.apply(lat, mix, out=y.view, ws=ws.view)
    assert y.intact() and ws.intact()
    assert torch.equal(y.view, dp.apply(lat, mix))
