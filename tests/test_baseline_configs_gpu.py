"""Parity at the BASELINE.json configurations themselves, against the CPU oracle.

Every check here runs the CUDA path at the exact benchmark shape (the GEMM instances,
tile schedules and workspace layouts the bench times) and compares a SUBSET of the
output with the fp64 oracle.  The subsets are exact pins, not samples of a tolerance:
the SHT loops per field (harmonics.hpp:139, :181), and both channel mixes are linear per
output row (convolution.hpp:207-218, :295-302), so output channel o depends only on
mix[o] / kernel[o] and on the full input.  The oracle side runs on all host cores
(reference headers in oracle/_ref where built, else the C restatement).
Bar: relative L2 <= 1e-5 (fp32 I/O, 3xTF32 tensor-core contractions).
"""
import math
import os
from concurrent.futures import ThreadPoolExecutor

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
DEV = torch.device("cuda", 0)
PI = math.pi
EQ, GA = 0, 1
THREADS = max(1, os.cpu_count() or 1)


def _pmap(fn, items):
    with ThreadPoolExecutor(min(THREADS, len(items))) as ex:
        return list(ex.map(fn, items))


def test_cfg2_bench_batch_fields_vs_oracle():
    """configs[1]: 721x1440 equiangular, lmax=721/mmax=720, F = 1024 fields -- the bench's
    own batch (its GEMM instance and tile schedule).  Fields 0, 511 and 1023 of the forward
    coefficients and of the round trip against the oracle; the whole batch must round-trip
    to the band-limited projection, which the oracle pins per field."""
    F = 1024
    g = S.build_equiangular(721, 1440)
    p = S.ShtPlan(g, 721, 720, "3xtf32", allow_equiangular_forward=True)
    sub = [0, 511, 1023]
    xs = {f: oracle.random_field((1, 721, 1440), 1 + f) for f in sub}
    x = torch.empty((F, 721, 1440), dtype=torch.float32, device=DEV)
    gen = torch.Generator(device=DEV).manual_seed(3)
    x.uniform_(-1, 1, generator=gen)
    for f in sub:
        x[f] = torch.tensor(xs[f][0], dtype=torch.float32, device=DEV)
    c = p.forward(x, L.SPH_LAYOUT_DENSE_LM)
    y = p.inverse(c, F, L.SPH_LAYOUT_DENSE_LM)
    torch.cuda.synchronize()

    def oracle_pair(f):
        ref = oracle.orc().sht_forward(EQ, 721, 1440, 721, 720, xs[f])
        return ref, oracle.orc().sht_inverse(EQ, 721, 1440, ref)

    refs = dict(zip(sub, _pmap(oracle_pair, sub)))
    for f in sub:
        cf = c[f].cpu().numpy().astype(np.float64)
        assert rel_l2(cf[..., 0] + 1j * cf[..., 1], refs[f][0][0]) <= TOL, f
        assert rel_l2(y[f].cpu().numpy(), refs[f][1][0]) <= TOL, f


def test_cfg3_bench_shape_channel_subset_vs_oracle():
    """configs[2] at the bench shape: DISCO 721x1440 eq -> 360x720 Gaussian, Morlet K=9,
    cutoff 3pi/360, 64 -> 256 channels, batch 4 (the BN=256 mix GEMM instance).  Output
    channels {0, 127, 255} of samples {0, 3} against the unmodified reference."""
    op = S.DiscoOperator(S.build_equiangular(721, 1440), S.build_gaussian(360, 720),
                         S.morlet_basis(3 * PI / 360))
    B, cin, cout = 4, 64, 256
    xs = [oracle.random_field((cin, 721, 1440), 1 + b) for b in range(B)]
    mix = oracle.random_field((cout, cin, 9), 77)
    y = op.apply(torch.tensor(np.stack(xs), dtype=torch.float32, device=DEV),
                 torch.tensor(mix, dtype=torch.float32, device=DEV))
    torch.cuda.synchronize()
    assert tuple(y.shape) == (B, cout, 360, 720)
    outs = [0, 127, 255]
    for b in (0, 3):
        if oracle.ref_available():
            _, _, ref = oracle.ref().bench_disco(EQ, 721, 1440, GA, 360, 720, 3 * PI / 360, xs[b],
                                                 mix[outs], THREADS, want_y=True)
        else:
            oop = oracle.orc().disco_assemble(EQ, 721, 1440, GA, 360, 720, 3 * PI / 360)
            ref = oracle.orc().disco_apply(oop, xs[b], mix[outs])
        got = y[b, outs].cpu().numpy().astype(np.float64)
        assert rel_l2(got, ref) <= TOL, b


def _sht_fields(kind, nlat, nlon, lmax, mmax, x):
    chunks = np.array_split(np.arange(x.shape[0]), min(THREADS, x.shape[0]))
    parts = _pmap(lambda ix: oracle.orc().sht_forward(kind, nlat, nlon, lmax, mmax, x[ix]), chunks)
    return np.concatenate(parts)


def test_cfg4_spectral_conv_c256_vs_oracle():
    """configs[3] global block conv: spectral_conv at 360x720 Gaussian, 256 -> 256 channels,
    klmax = 360 (convolution.hpp:286-304).  Output channels {0, 255}: the oracle's forward
    SHT of all 256 inputs, the per-degree mix of those two rows (:295-302), its inverse."""
    g = S.build_gaussian(360, 720)
    C = 256
    x = oracle.random_field((C, 360, 720), 41)
    k = oracle.random_field((C, C, 360), 42) / 16.0
    y = S.spectral_conv(S.SphericalField(g, torch.tensor(x[None], dtype=torch.float32, device=DEV)),
                        torch.tensor(k, dtype=torch.float32, device=DEV)).data
    torch.cuda.synchronize()
    cx = _sht_fields(GA, 360, 720, 360, 360, x)                  # [C][360][360]
    outs = [0, 255]
    mixed = np.einsum("oil,ilm->olm", k[outs], cx)
    ref = np.stack([oracle.orc().sht_inverse(GA, 360, 720, mixed[i:i + 1])[0] for i in range(len(outs))])
    got = y[0, outs].cpu().numpy().astype(np.float64)
    assert rel_l2(got, ref) <= TOL


def test_cfg4_local_block_disco_c256_vs_oracle():
    """configs[3] local block conv: DISCO 360x720 -> 360x720 Gaussian (stride 1), Morlet
    cutoff 3pi/360, 256 -> 256 channels.  Output channels {0, 128, 255} against the
    unmodified reference."""
    g = S.build_gaussian(360, 720)
    op = S.DiscoOperator(g, g, S.morlet_basis(3 * PI / 360))
    C = 256
    x = oracle.random_field((C, 360, 720), 43)
    mix = oracle.random_field((C, C, 9), 44) / 48.0
    y = op.apply(torch.tensor(x[None], dtype=torch.float32, device=DEV),
                 torch.tensor(mix, dtype=torch.float32, device=DEV))
    torch.cuda.synchronize()
    outs = [0, 128, 255]
    if oracle.ref_available():
        _, _, ref = oracle.ref().bench_disco(GA, 360, 720, GA, 360, 720, 3 * PI / 360, x, mix[outs],
                                             THREADS, want_y=True)
    else:
        oop = oracle.orc().disco_assemble(GA, 360, 720, GA, 360, 720, 3 * PI / 360)
        ref = oracle.orc().disco_apply(oop, x, mix[outs])
    assert rel_l2(y[0, outs].cpu().numpy().astype(np.float64), ref) <= TOL
