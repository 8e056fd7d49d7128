"""Multi-process worker for the NCCL product path of the distributed SHT / DISCO
(csrc/dist.cu through paper_2507_12144_b200.dist.NcclComm / DistShtPlan / DistDiscoPlan),
launched by tests/test_dist.py with torchrun on >= 2 GPUs.

Every rank computes its block through the C ABI; the blocks are gathered on every rank
and compared with the fp64 oracle run serially on the whole field (the reference's
dist_sht_forward 1x1 == serial equivalence, distsim.hpp:404-463, and serial sht_inverse /
disco_apply for the mirrored inverse and Alg. 2).  Rank 0 writes a JSON report.
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
import paper_2507_12144_b200 as S  # noqa: E402
from paper_2507_12144_b200 import dist as D  # noqa: E402

PI = math.pi
EQ, GA = 0, 1


def gather_blocks(local, r0, r1, shape):
    """Assemble the global [C, A, B, ...] tensor from every rank's block at rows r0 / cols r1."""
    objs = [None] * dist.get_world_size()
    dist.all_gather_object(objs, (local.detach().cpu().numpy().astype(np.float64), r0, r1))
    out = np.zeros(shape)
    for blk, a, b in objs:
        out[:, a:a + blk.shape[1], b:b + blk.shape[2]] = blk
    return out


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def check_sht(comm, dev, kind, nlat, nlon, lmax, mmax, C, seed, subset=None):
    grid = S.build_equiangular(nlat, nlon) if kind == EQ else S.build_gaussian(nlat, nlon)
    plan = D.DistShtPlan(comm, grid, lmax, mmax, C)
    x = oracle.random_field((C, nlat, nlon), seed)
    xl = plan.shard(torch.tensor(x, dtype=torch.float32, device=dev))
    c = plan.forward(xl)
    y = plan.inverse(c)
    torch.cuda.synchronize()
    cg = gather_blocks(c, plan.l0, plan.m0, (C, lmax, mmax, 2))
    yg = gather_blocks(y, plan.h0, plan.w0, (C, nlat, nlon))
    if dist.get_rank() != 0:  # the serial oracle runs once, on rank 0
        return None
    sub = list(range(C)) if subset is None else subset
    ref = oracle.orc().sht_forward(kind, nlat, nlon, lmax, mmax, x[sub])
    yref = oracle.orc().sht_inverse(kind, nlat, nlon, ref)
    got = cg[sub, ..., 0] + 1j * cg[sub, ..., 1]
    # the inverse of the gathered forward: the mirrored Alg. 1 against serial sht_inverse
    return rel(got, ref), rel(yg[sub], yref)


def check_disco(comm, dev, ik, ih, iw, ok, oh, ow, cut, cin, cout, seed, outs=None):
    gi = S.build_equiangular(ih, iw) if ik == EQ else S.build_gaussian(ih, iw)
    go = S.build_equiangular(oh, ow) if ok == EQ else S.build_gaussian(oh, ow)
    op = S.DiscoOperator(gi, go, S.morlet_basis(cut), device=dev)
    plan = D.DistDiscoPlan(comm, op, cin, cout)
    x = oracle.random_field((cin, ih, iw), seed)
    mix = oracle.random_field((cout, cin, 9), seed + 1)
    y = plan.apply(plan.shard(torch.tensor(x, dtype=torch.float32, device=dev)),
                   torch.tensor(mix, dtype=torch.float32, device=dev))
    torch.cuda.synchronize()
    yg = gather_blocks(y, plan.ho0, plan.wo0, (cout, oh, ow))
    if dist.get_rank() != 0:
        return None
    outs = list(range(cout)) if outs is None else outs
    if oracle.ref_available():
        _, _, ref = oracle.ref().bench_disco(ik, ih, iw, ok, oh, ow, cut, x, mix[outs], os.cpu_count() or 1,
                                             want_y=True)
    else:
        oop = oracle.orc().disco_assemble(ik, ih, iw, ok, oh, ow, cut)
        ref = oracle.orc().disco_apply(oop, x, mix[outs])
    return rel(yg[outs], ref)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nh", type=int, required=True)
    ap.add_argument("--nw", type=int, required=True)
    ap.add_argument("--big", type=int, default=0, help="also the 721x1440 (configs[4]) grids")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = D.NcclComm(D.CommGrid((1, 1, args.nh, args.nw)))
    rep = {}
    # Gaussian 16x32 (test_distsim.cpp:166-186 grid), 5 channels: uneven channel slices
    rep["sht_ga16"] = check_sht(comm, dev, GA, 16, 32, 16, 16, 5, 30)
    # cfg1 grid (equiangular 91x180, lmax 91 / mmax 90), 3 channels: with 4 ranks one
    # rank computes no channel at all
    rep["sht_eq91"] = check_sht(comm, dev, EQ, 91, 180, 91, 90, 3, 1)
    # traffic: 2 plane all-to-alls per direction (the reference's 4 per-axis ones, fused)
    csv = comm.traffic_csv()
    rep["traffic_csv"] = csv
    rows = [ln.split(",") for ln in csv.strip().splitlines()[1:]]
    rep["sht_calls"] = {r[0]: int(r[4]) for r in rows}
    # DISCO Gaussian 16x32 -> 8x16 (test_distsim.cpp:204-228), odd latitude count 9x16
    rep["disco_ga16"] = check_disco(comm, dev, GA, 16, 32, GA, 8, 16, 3 * PI / 8, 3, 2, 33)
    rep["disco_eq9"] = check_disco(comm, dev, EQ, 9, 16, EQ, 9, 16, 3 * PI / 9, 2, 1, 35)
    rep["disco_eq91"] = check_disco(comm, dev, EQ, 91, 180, GA, 45, 90, 3 * PI / 45, 5, 3, 37)
    if args.big:
        # configs[4] grids: 721x1440 equiangular, lmax 721 / mmax 720 (8 channels, fields 0
        # and 7 against the oracle), DISCO -> 360x720 Gaussian (16 -> 4 channels, outputs 0, 3)
        rep["sht_721"] = check_sht(comm, dev, EQ, 721, 1440, 721, 720, 8, 51, subset=[0, 7])
        rep["disco_721"] = check_disco(comm, dev, EQ, 721, 1440, GA, 360, 720, 3 * PI / 360, 16, 4, 53,
                                       outs=[0, 3])
    if dist.get_rank() == 0:
        with open(args.out, "w") as f:
            json.dump(rep, f)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
