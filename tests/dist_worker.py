"""Multi-process worker for the distributed SHT / DISCO tests (launched by
tests/test_dist.py through ``torch.distributed.run`` with 127.0.0.1 rendezvous).

--device cpu  : gloo collectives + an fp64 ORACLE compute backend (test infrastructure
                only) -> checks the host logic (canonical splits, transposes, halo,
                reduce-scatter, traffic bookkeeping) bit-for-bit-ish against the
                reference simulator's golden outputs.
--device cuda : NCCL collectives + the product GpuBackend (libsphgpu.so kernels).
Rank 0 writes a JSON report to --out.
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2507_12144_b200 import dist as D  # noqa: E402

PI = math.pi


class _Grid:
    def __init__(self, kind, nlat, nlon):
        self.kind, self.nlat, self.nlon = kind, nlat, nlon


class OracleBackend:
    """fp64 CPU stand-in for GpuBackend (tests only): the reference arithmetic of
    distsim.hpp:413-430 (rfft_bins * 2pi/nlon) and :437-459 (weighted table, global m)."""

    def fft_stage(self, grid, lmax, mmax, x):
        o = oracle.orc()
        xn = x.numpy()
        out = np.zeros(xn.shape[:2] + (mmax, 2))
        for c in range(xn.shape[0]):
            for h in range(xn.shape[1]):
                b = o.rfft_bins(xn[c, h], mmax) * (2 * PI / grid.nlon)
                out[c, h, :, 0], out[c, h, :, 1] = b.real, b.imag
        return torch.from_numpy(out)

    def sht_full(self, grid, lmax, mmax, x):
        """The fused order's per-rank transform (dist.py: _dist_sht_fused): all latitudes
        and longitudes of the rank's channel slice -> [C, lmax, mmax, 2], the reference's
        Alg. 1 arithmetic on one rank (dist_sht_forward 1x1 == the C restatement)."""
        xn = x.numpy()
        c = oracle.orc().sht_forward(grid.kind, grid.nlat, grid.nlon, lmax, mmax, xn) if xn.shape[0] else \
            np.zeros((0, lmax, mmax), complex)
        return torch.from_numpy(np.stack([c.real, c.imag], -1))

    def legendre_stage(self, grid, lmax, mmax, bins, m0):
        o = oracle.orc()
        colat, w = o.grid(grid.kind, grid.nlat, grid.nlon)
        tab = o.legendre_table(lmax, mmax, colat) * (w * grid.nlon / (2 * PI))[:, None, None]
        b = bins.numpy()
        G = b[..., 0] + 1j * b[..., 1]                      # [C, nlat, mloc]
        mloc = G.shape[2]
        out = np.zeros((G.shape[0], lmax, mloc, 2))
        for ml in range(mloc):
            m = m0 + ml
            T = tab[:, :, m]                                # [nlat, lmax]
            acc = np.einsum("il,ci->cl", T, G[:, :, ml])
            acc[:, :m] = 0
            out[:, :, ml, 0], out[:, :, ml, 1] = acc.real, acc.imag
        return torch.from_numpy(out)

    def weighted_crps(self, f, o, w, variant):
        """distsim.hpp:598-616 with crps_pointwise (metrics.hpp:160-209), fp64."""
        fn, on = f.numpy(), o.numpy()
        E, C, ns = fn.shape
        out = np.zeros(C)
        n = float(E)
        for c in range(C):
            acc = 0.0
            for k in range(ns):
                u = np.sort(fn[:, c, k])
                ob = on[c, k]
                if variant == "cdf":
                    e = np.arange(1, E + 1)
                    v = np.where(u <= ob, (2 * e - 1) / (n * n) * (ob - u), (2 * n + 1 - 2 * e) / (n * n) * (u - ob)).sum()
                else:
                    skill = np.abs(u - ob).sum() / n
                    pair = 2.0 * ((2 * np.arange(1, E + 1) - 1 - n) * u).sum()
                    denom = 2 * n * (n - 1) if variant == "fair" else 2 * n * n
                    v = skill - pair / denom
                acc += w[k] * v
            out[c] = acc / (4 * PI)
        return torch.from_numpy(out)

    def disco_rows(self, op, x, h_in0, ho0, nout, mix):
        xn = x.numpy()
        full = np.zeros((xn.shape[0], op.in_grid.nlat, op.in_grid.nlon))
        full[:, h_in0:h_in0 + xn.shape[1]] = xn
        y = oracle.orc().disco_apply(op.oop, full, mix.numpy())
        return torch.from_numpy(np.ascontiguousarray(y[:, ho0:ho0 + nout]))


class OracleDiscoOp:
    def __init__(self, ik, ih, iw, ok, oh, ow, cut):
        self.in_grid, self.out_grid = _Grid(ik, ih, iw), _Grid(ok, oh, ow)
        self.oop = oracle.orc().disco_assemble(ik, ih, iw, ok, oh, ow, cut)
        rp, hi = self.oop["row_ptr"], self.oop["h_in"]
        self.bands = [(int(hi[rp[h]:rp[h + 1]].min()), int(hi[rp[h]:rp[h + 1]].max()) + 1)
                      for h in range(oh)]

    def input_rows(self, ho0, nout):
        lo = min(self.bands[h][0] for h in range(ho0, ho0 + nout))
        hi = max(self.bands[h][1] for h in range(ho0, ho0 + nout))
        return lo, hi - lo


def run_crps(args, cuda, dev, G):
    """dist_crps (Alg. 3) vs the serial crps_field (test_distsim.cpp:250-300)."""
    ctx = D.DistContext(D.CommGrid((args.nb, args.ne, args.nh, args.nw)))
    rep = {}
    # batch item b scores the golden sample scaled by (1 + b): CRPS is positively
    # homogeneous, so its score is (1 + b) * golden -- a rank that mixed in another batch
    # item's partial sums would be off by a whole sample's score.
    scale = 1.0 + ctx.index(D.BATCH)
    for key, nlat, nlon in (("crps_ga8_E8", 8, 16), ("crps_ga5_E8", 5, 8)):
        ens, obs, want = G[key + "_ens"] * scale, G[key + "_obs"] * scale, G[key] * scale
        E = ens.shape[0]
        ep = D.canonical_split(E, args.ne)
        hp, wp = D.canonical_split(nlat, args.nh), D.canonical_split(nlon, args.nw)
        e, i, j = ctx.index(D.ENSEMBLE), ctx.index(D.POLAR), ctx.index(D.AZIMUTH)
        fl = ens[D.split_offset(ep, e):D.split_offset(ep, e) + ep[e], :,
                 D.split_offset(hp, i):D.split_offset(hp, i) + hp[i],
                 D.split_offset(wp, j):D.split_offset(wp, j) + wp[j]]
        ol = obs[:, D.split_offset(hp, i):D.split_offset(hp, i) + hp[i],
                 D.split_offset(wp, j):D.split_offset(wp, j) + wp[j]]
        dt = torch.float32 if cuda else torch.float64
        f = D.Sharded(torch.tensor(np.ascontiguousarray(fl), dtype=dt, device=dev), {0: ep, 2: hp, 3: wp})
        o = D.Sharded(torch.tensor(np.ascontiguousarray(ol), dtype=dt, device=dev), {1: hp, 2: wp})
        if cuda:
            import paper_2507_12144_b200 as S
            grid, backend = S.build_gaussian(nlat, nlon), D.GpuBackend()
        else:
            backend = OracleBackend()
            colat, w = oracle.orc().grid(1, nlat, nlon)
            grid = _Grid(1, nlat, nlon)
            grid.quad_weights = w
        ctx.log = D.TrafficLog()
        got = D.dist_crps(ctx, f, o, grid, "fair", backend).cpu().numpy()
        err = torch.tensor([float(np.abs(got - want).max() / max(1.0, np.abs(want).max()))],
                           dtype=torch.float64, device=dev)
        dist.all_reduce(err, op=dist.ReduceOp.MAX)   # worst rank, every batch item
        rep[key] = float(err.item())
        rep[key + "_calls"] = {c: ctx.log.calls("dist_crps", c) for c in ("all_to_all", "scatter", "all_reduce")}
    return rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ne", type=int, default=0, help="dist_crps mode with this many ensemble ranks")
    ap.add_argument("--nb", type=int, default=1, help="dist_crps: batch ranks")
    ap.add_argument("--device", default="cpu")
    ap.add_argument("--nh", type=int, required=True)
    ap.add_argument("--nw", type=int, required=True)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    cuda = args.device == "cuda"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if cuda:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dev = torch.device("cuda", local)
    else:
        dist.init_process_group("gloo")
        dev = torch.device("cpu")
    G = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    if args.ne:
        rep = run_crps(args, cuda, dev, G)
        if dist.get_rank() == 0:
            with open(args.out, "w") as f:
                json.dump(rep, f)
        dist.barrier()
        dist.destroy_process_group()
        return
    ctx = D.DistContext(D.CommGrid((1, 1, args.nh, args.nw)))
    rep = {}
    dt = torch.float32 if cuda else torch.float64

    # ---- distributed SHT, Gaussian 16x32, lmax = mmax = 16 (test_distsim.cpp:166-186)
    if cuda:
        import paper_2507_12144_b200 as S
        grid = S.build_gaussian(16, 32)
        backend = D.GpuBackend()
    else:
        grid, backend = _Grid(1, 16, 32), OracleBackend()
    x = torch.tensor(oracle.random_field((3, 16, 32), 30), dtype=dt, device=dev)
    out = D.dist_sht_forward(ctx, D.shard_field(ctx, x), grid, 16, 16, backend, order="reference")
    glob = D.unshard(ctx, out).cpu().numpy()
    got = glob[..., 0] + 1j * glob[..., 1]
    key = f"dist_sht_{args.nh}x{args.nw}"
    want = G[key] if key in G.files else oracle.orc().sht_forward(1, 16, 32, 16, 16, x.cpu().numpy())
    rep["sht_err"] = float(np.abs(got - want).max() / np.abs(want).max())
    rep["sht_a2a_calls"] = ctx.log.calls("dist_sht", "all_to_all")
    rep["sht_csv"] = ctx.log.csv()
    if key + "_csv" in G.files:
        rep["ref_sht_csv"] = str(G[key + "_csv"])

    # ---- fused order (T1, T3', per-rank SHT, T4', T2'), pipelined over 3 channel chunks,
    # on both backends: the oracle's sht_full makes the order testable over gloo
    x = torch.tensor(oracle.random_field((7, 16, 32), 36), dtype=dt, device=dev)
    out = D.dist_sht_forward(ctx, D.shard_field(ctx, x), grid, 16, 16, backend, chunks=3)
    glob = D.unshard(ctx, out).cpu().numpy()
    got = glob[..., 0] + 1j * glob[..., 1]
    want = oracle.orc().sht_forward(1, 16, 32, 16, 16, x.cpu().numpy())
    rep["sht_chunked_err"] = float(np.abs(got - want).max() / np.abs(want).max())

    # ---- equiangular 91x180 (cfg1 grid) dist SHT vs the oracle (reference equiangular path)
    if cuda:
        grid = S.build_equiangular(91, 180)
    else:
        grid = _Grid(0, 91, 180)
    x = torch.tensor(oracle.random_field((4, 91, 180), 1), dtype=dt, device=dev)
    out = D.dist_sht_forward(ctx, D.shard_field(ctx, x), grid, 91, 90, backend)
    glob = D.unshard(ctx, out).cpu().numpy()
    got = glob[..., 0] + 1j * glob[..., 1]
    want = G["cfg1_fwd"]
    rep["sht_eq_rel"] = float(np.linalg.norm(got - want) / np.linalg.norm(want))

    # ---- distributed DISCO, Gaussian 16x32 -> 8x16 (test_distsim.cpp:204-228)
    if cuda:
        op = S.DiscoOperator(S.build_gaussian(16, 32), S.build_gaussian(8, 16), S.morlet_basis(3 * PI / 8))
    else:
        op = OracleDiscoOp(1, 16, 32, 1, 8, 16, 3 * PI / 8)
    mix = torch.tensor(oracle.random_field((2, 3, 9), 32), dtype=dt, device=dev)
    x = torch.tensor(oracle.random_field((3, 16, 32), 33), dtype=dt, device=dev)
    ctx.log = D.TrafficLog()
    y = D.dist_disco_apply(ctx, D.shard_field(ctx, x), op, mix, backend)
    glob = D.unshard(ctx, y).cpu().numpy()
    key = f"dist_disco_{args.nh}x{args.nw}"
    if key in G.files:
        want = G[key]
    else:
        oop = oracle.orc().disco_assemble(1, 16, 32, 1, 8, 16, 3 * PI / 8)
        want = oracle.orc().disco_apply(oop, x.cpu().numpy(), mix.cpu().numpy())
    rep["disco_err"] = float(np.abs(glob - want).max() / np.abs(want).max())
    rep["disco_csv"] = ctx.log.csv()
    rep["disco_calls"] = {c: ctx.log.calls("dist_disco", c) for c in ("all_to_all", "halo", "reduce_scatter")}

    # ---- odd latitude count over the polar axis (test_distsim.cpp:230-248)
    if args.nh == 2:
        if cuda:
            op = S.DiscoOperator(S.build_equiangular(9, 16), S.build_equiangular(9, 16), S.morlet_basis(3 * PI / 9))
        else:
            op = OracleDiscoOp(0, 9, 16, 0, 9, 16, 3 * PI / 9)
        mix = torch.tensor(oracle.random_field((1, 2, 9), 34), dtype=dt, device=dev)
        x = torch.tensor(oracle.random_field((2, 9, 16), 35), dtype=dt, device=dev)
        sh = D.shard_field(ctx, x)
        rep["odd_split"] = sh.split[1]
        y = D.unshard(ctx, D.dist_disco_apply(ctx, sh, op, mix, backend)).cpu().numpy()
        oop = oracle.orc().disco_assemble(0, 9, 16, 0, 9, 16, 3 * PI / 9)
        want = oracle.orc().disco_apply(oop, x.cpu().numpy(), mix.cpu().numpy())
        rep["odd_err"] = float(np.abs(y - want).max() / np.abs(want).max())

    if dist.get_rank() == 0:
        with open(args.out, "w") as f:
            json.dump(rep, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
