"""Generate the golden vectors in tests/golden/golden.npz from the UNMODIFIED reference.

Runs only where /root/reference exists (it drives oracle/_ref/libsphref.so, the
reference headers compiled behind oracle/ref_driver.cpp).  Inputs are the reference
test-suite RNG stream (proj/tests/oracles.hpp:105-112: mt19937_64 + U(-1,1)), so
every fixture stores its seed; outputs are the reference's fp64 results.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

EQ, GA = oracle.EQUIANGULAR, oracle.GAUSSIAN
PI = np.pi


def main():
    r = oracle.ref()
    G = {}

    # RNG stream (oracles.hpp:105-112)
    G["rng_seed1"] = r.random_uniform((64,), 1)

    # grids (grid.hpp:69-128; test_grid.cpp pins)
    for kind, nlat, nlon in [(EQ, 9, 16), (EQ, 91, 180), (EQ, 721, 1440), (GA, 16, 32),
                             (GA, 6, 12), (GA, 360, 720), (GA, 1, 4)]:
        c, w = r.grid(kind, nlat, nlon)
        G[f"grid_{kind}_{nlat}_{nlon}_colat"] = c
        G[f"grid_{kind}_{nlat}_{nlon}_w"] = w

    # rfft_bins (fft.hpp:97) on the lengths the hot path uses + test_fft.cpp lengths
    for n in [1, 2, 3, 5, 7, 12, 16, 20, 33, 90, 180, 720, 1440]:
        x = r.random_uniform((n,), 1000 + n)
        G[f"rfft_{n}"] = r.rfft_bins(x, n // 2 + 1)

    # Legendre tables (harmonics.hpp:59 / :106)
    G["leg_eq_9_16_w"] = r.legendre_table(9, 8, EQ, 9, 16, weighted=True)
    G["leg_ga_16_32"] = r.legendre_table(16, 16, GA, 16, 32, weighted=False)

    # SHT cfg1: 91x180 equiangular, lmax=91, mmax=90; 4-channel subset of the seed-1
    # 32-channel field (the reference loops per channel, harmonics.hpp:139, so the
    # subset is exact).  Forward = dist_sht_forward 1x1 (the reference's equiangular path).
    x = r.random_uniform((32, 91, 180), 1)
    c = r.sht_forward(EQ, 91, 180, 91, 90, x[:4])
    G["cfg1_fwd"] = c
    G["cfg1_rt"] = r.sht_inverse(EQ, 91, 180, c)

    # Gaussian round trip 32x64 (test_harmonics.cpp:116-131 / acceptance c1 shape)
    x = r.random_uniform((2, 32, 64), 7)
    c = r.sht_forward(GA, 32, 64, 32, 32, x)
    G["ga32_fwd"] = c
    G["ga32_rt"] = r.sht_inverse(GA, 32, 64, c)
    # Gaussian 16x32 mode truncation (test_distsim.cpp:188-202)
    x = r.random_uniform((2, 16, 32), 31)
    G["ga16_m8_fwd"] = r.sht_forward(GA, 16, 32, 16, 8, x)
    # equiangular odd sizes (uneven pole handling), 9x16 (test_harmonics.cpp:102)
    x = r.random_uniform((3, 9, 16), 5)
    c = r.sht_forward(EQ, 9, 16, 9, 8, x)
    G["eq9_fwd"] = c
    G["eq9_rt"] = r.sht_inverse(EQ, 9, 16, c)
    # inverse on a grid with fewer longitudes than 2*mmax (msynth clamp, harmonics.hpp:179)
    cf = r.random_uniform((1, 8, 8, 2), 8)
    cf = cf[..., 0] + 1j * cf[..., 1]
    G["inv_msynth"] = r.sht_inverse(EQ, 9, 10, cf)

    # DISCO (convolution.hpp:141-220, 226-266); mixes from random_mix semantics
    # (test_convolution.cpp:76-82)
    cases = {
        "ga16_ga8": (GA, 16, 32, GA, 8, 16, 3 * PI / 8, 3, 2),
        "eq16_eq16": (EQ, 16, 32, EQ, 16, 32, 4 * PI / 16, 3, 2),
        "eq12_stride3": (EQ, 12, 24, EQ, 12, 8, 3 * PI / 12, 1, 1),
        "eq91_ga45": (EQ, 91, 180, GA, 45, 90, 3 * PI / 45, 4, 8),
        "eq9_eq9": (EQ, 9, 16, EQ, 9, 16, 3 * PI / 9, 2, 1),
    }
    for name, (ik, ih, iw, ok, oh, ow, cut, cin, cout) in cases.items():
        rows, K, hh, ww, vv, bb = r.disco_entries(ik, ih, iw, ok, oh, ow, cut)
        mix = r.random_uniform((cout, cin, K), 77)
        x = r.random_uniform((cin, ih, iw), 78)
        G[f"disco_{name}_rows"] = rows
        G[f"disco_{name}_y"] = r.disco_apply(ik, ih, iw, ok, oh, ow, cut, x, mix)
        v = r.random_uniform((cout, oh, ow), 79)
        G[f"disco_{name}_yT"] = r.disco_transpose_apply(ik, ih, iw, ok, oh, ow, cut, v, mix)
    # isotropic basis (K = 1) one-cell cutoff (test_convolution.cpp:153-163)
    x = r.random_uniform((1, 12, 24), 5)
    G["disco_iso_eq12_y"] = r.disco_apply(EQ, 12, 24, EQ, 12, 24, PI / 12, x,
                                          np.ones((1, 1, 1)), basis=1)
    # cfg3 row structure (721x1440 eq -> 360x720 Gaussian, cutoff 3pi/360)
    rows, K = r.disco_rows(EQ, 721, 1440, GA, 360, 720, 3 * PI / 360)
    G["disco_cfg3_rows"] = rows

    # spectral conv (convolution.hpp:286)
    x = r.random_uniform((3, 16, 32), 55)
    k = r.random_uniform((2, 3, 12), 56)
    G["sconv_ga16_y"] = r.spectral_conv(GA, 16, 32, k, x)

    # block_apply (model.hpp:337-370): levels 1, embed 8 -> C = 16, cond 8, hidden 32
    C_, Cc, H = 16, 8, 32
    for glob in (0, 1):
        x = r.random_uniform((C_, 16, 32), 90)
        cond = r.random_uniform((Cc, 16, 32), 91)
        convw = r.random_uniform((C_, C_ + Cc, 16 if glob else 9), 92) * 0.2
        w1 = r.random_uniform((H, C_), 93) * 0.3
        b1 = r.random_uniform((H,), 94) * 0.1
        w2 = r.random_uniform((C_, H), 95) * 0.3
        b2 = r.random_uniform((C_,), 96) * 0.1
        sc = r.random_uniform((C_,), 97)
        G[f"block_g{glob}_y"] = r.block_apply(16, 32, 1, 8, H, glob, 3 * PI / 16, 16, x, cond,
                                              convw, w1, b1, w2, b2, sc)

    # distributed (distsim.hpp:404, :468) -- outputs and traffic CSV
    x = r.random_uniform((3, 16, 32), 30)
    for nh, nw in [(2, 4), (1, 2), (2, 1), (4, 2)]:
        out, csv = r.dist_sht_forward(GA, 16, 32, 16, 16, x, nh, nw)
        G[f"dist_sht_{nh}x{nw}"] = out
        G[f"dist_sht_{nh}x{nw}_csv"] = np.array(csv)
    x = r.random_uniform((3, 16, 32), 33)
    mix = r.random_uniform((2, 3, 9), 32)
    for nh, nw in [(2, 2), (2, 1), (1, 2)]:
        y, csv = r.dist_disco_apply(GA, 16, 32, GA, 8, 16, 3 * PI / 8, x, mix, nh, nw)
        G[f"dist_disco_{nh}x{nw}"] = y
        G[f"dist_disco_{nh}x{nw}_csv"] = np.array(csv)

    # bilinear_resample with pole extension (resample.hpp:20-114; test_resample.cpp:12-123)
    rcases = {
        "ga8_eq13": (GA, 8, 16, 0, EQ, 13, 20),     # constants / range case
        "eq9_ga7": (EQ, 9, 12, 0, GA, 7, 9),        # four-weight formula case
        "eq4_eq4x6": (EQ, 4, 4, 0, EQ, 4, 6),       # longitude wrap-around
        "ga8_id": (GA, 8, 16, 0, GA, 8, 16),        # identity
        "eq9_id": (EQ, 9, 16, 0, EQ, 9, 16),
        "p2p4": (EQ, 4, 4, 1, EQ, 5, 8),            # input already touching both poles
        "eq91_ga45": (EQ, 91, 180, 0, GA, 45, 90),
        "ga45_eq91": (GA, 45, 90, 0, EQ, 91, 180),  # decoder direction (Gaussian -> eq)
    }
    for name, (ik, ih, iw, lp, ok, oh, ow) in rcases.items():
        x = r.random_uniform((2, ih, iw), 40)
        G[f"resample_{name}"] = r.bilinear_resample(ik, ih, iw, ok, oh, ow, x, in_last_pi=lp)

    # spectral_resample (resample.hpp:120-132): Gaussian / equiangular inputs, up and down
    for name, (ik, ih, iw, ok, oh, ow) in {"ga8_ga12": (GA, 8, 16, GA, 12, 24),
                                           "ga12_eq9": (GA, 12, 24, EQ, 9, 16),
                                           "eq9_ga8": (EQ, 9, 16, GA, 8, 16),
                                           "ga45_eq91": (GA, 45, 90, EQ, 91, 180)}.items():
        x = r.random_uniform((2, ih, iw), 41)
        G[f"sresample_{name}"] = r.spectral_resample(ik, ih, iw, ok, oh, ow, x)

    # decoder group (model.hpp:372-394): disco_apply(dec_op, bilinear_resample(latent, out))
    dcases = {
        "ga8_eq17": (GA, 8, 16, EQ, 17, 32, 3 * PI / 16, 3, 2),    # r = 2, both poles extended
        "ga6_ga12": (GA, 6, 12, GA, 12, 36, 3 * PI / 12, 2, 3),    # r = 3, Gaussian -> Gaussian
        "eq5_eq9": (EQ, 5, 8, EQ, 9, 16, 3 * PI / 9, 2, 1),        # latent touches the north pole
        "eq9_eq9x24": (EQ, 9, 16, EQ, 9, 24, 3 * PI / 9, 2, 2),    # ratio 1.5: unfused path
        "ga45_eq91": (GA, 45, 90, EQ, 91, 180, 3 * PI / 90, 4, 1),
    }
    for name, (lk, lh, lw, ok, oh, ow, cut, cin, cout) in dcases.items():
        lat = r.random_uniform((cin, lh, lw), 90)
        up = r.bilinear_resample(lk, lh, lw, ok, oh, ow, lat)
        mix = r.random_uniform((cout, cin, 9), 91)
        G[f"decoder_{name}_latent"] = lat
        G[f"decoder_{name}_mix"] = mix
        G[f"decoder_{name}_y"] = r.disco_apply(ok, oh, ow, ok, oh, ow, cut, up, mix)

    # SHT consumers (metrics.hpp:300-314 angular_psd, loss.hpp:37-81 spectral_crps_loss)
    x = r.random_uniform((3, 16, 32), 60)
    G["psd_ga16"] = r.angular_psd(GA, 16, 32, x)
    x = r.random_uniform((2, 45, 90), 61)
    G["psd_ga45"] = r.angular_psd(GA, 45, 90, x)
    ens = r.random_uniform((5, 2, 16, 32), 62)
    obs = r.random_uniform((2, 16, 32), 63)
    for v in range(3):
        G[f"scrps_ga16_v{v}"] = r.spectral_crps_loss(GA, 16, 32, ens, obs, 0, v)
    ens = r.random_uniform((8, 3, 45, 90), 64)
    obs = r.random_uniform((3, 45, 90), 65)
    G["scrps_ga45_v2_l20"] = r.spectral_crps_loss(GA, 45, 90, ens, obs, 20, 2)

    # noise_field synthesis (noise.hpp:95-97) of the reference's own AR(1) noise states
    kts = np.array([3.08e-5, 1.97e-3, 1.26e-1])
    f, c = r.noise_stream(GA, 24, 48, 24, kts, 1234, 3)
    G["noise_ga24_field"], G["noise_ga24_coeffs"] = f, c
    f, c = r.noise_stream(EQ, 33, 64, 32, kts, 99, 2)
    G["noise_eq33_field"], G["noise_eq33_coeffs"] = f, c

    # dist_crps targets: the serial crps_field (test_distsim.cpp:250-300)
    ens = r.random_uniform((8, 2, 8, 16), 66)
    obs = r.random_uniform((2, 8, 16), 67)
    G["crps_ga8_E8"], G["crps_ga8_E8_ens"], G["crps_ga8_E8_obs"] = r.crps_field(GA, 8, 16, ens, obs, 2), ens, obs
    ens = r.random_uniform((8, 1, 5, 8), 68)
    obs = r.random_uniform((1, 5, 8), 69)
    G["crps_ga5_E8"], G["crps_ga5_E8_ens"], G["crps_ga5_E8_obs"] = r.crps_field(GA, 5, 8, ens, obs, 2), ens, obs

    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(out, **G)
    print("wrote", out, os.path.getsize(out), "bytes,", len(G), "arrays")


if __name__ == "__main__":
    main()
