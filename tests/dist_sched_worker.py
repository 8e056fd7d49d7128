"""CPU (gloo) executor of the library's OWN distributed schedules (tests/test_dist.py).

The product distributed SHT / DISCO (csrc/dist.cu) runs a host-side layout
(csrc/dist_layout.hpp) that decides every rank's ranges, every all-to-all's counts and
offsets and every pack / unpack box.  libsphgpu.so exports that layout without a GPU
(sph_dist_sht_describe / sph_dist_disco_describe); this worker runs it over gloo with
numpy copies and the fp64 oracle as the local transform, then checks the gathered result
against the serial oracle to 1e-12.  The coefficient payload format (the stored triangle
m <= l of each (l, m) block, dist_layout.hpp) is restated here from its specification.
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
EQ, GA = 0, 1


def xchg(send, sched, P):
    sc, so, rc, ro = (sched[k * P:(k + 1) * P] for k in range(4))
    inp = torch.from_numpy(np.concatenate([send[so[p]:so[p] + sc[p]] for p in range(P)]).astype(np.float64))
    out = torch.empty(int(sum(rc)), dtype=torch.float64)
    dist.all_to_all_single(out, inp, output_split_sizes=list(rc), input_split_sizes=list(sc))
    recv = np.zeros(max([ro[p] + rc[p] for p in range(P)] + [0]))
    pos = 0
    for p in range(P):
        recv[ro[p]:ro[p] + rc[p]] = out.numpy()[pos:pos + rc[p]]
        pos += rc[p]
    return recv


def run_boxes(boxes, src, dst):
    for k in range(0, len(boxes), 9):
        so, do, n0, n1, n2, s0, s1, d0, d1 = boxes[k:k + 9]
        for a in range(n0):
            for b in range(n1):
                dst[do + a * d0 + b * d1:do + a * d0 + b * d1 + n2] = src[so + a * s0 + b * s1:so + a * s0 + b * s1 + n2]


def gather(block, r0, r1, shape):
    objs = [None] * dist.get_world_size()
    dist.all_gather_object(objs, (block, r0, r1))
    out = np.zeros(shape, dtype=block.dtype)
    for blk, a, b in objs:
        out[:, a:a + blk.shape[1], b:b + blk.shape[2]] = blk
    return out


def sht_case(nh, nw, q, kind, nlat, nlon, lmax, mmax, C, seed):
    P = nh * nw
    d = lambda what, r=q: D.describe_sht(nh, nw, r, nlat, nlon, lmax, mmax, C, what)  # noqa: E731
    o = oracle.orc()
    x = oracle.random_field((C, nlat, nlon), seed)
    h0, hn, w0, wn, l0, ln, m0, mn, c0, cn = d(0)
    rng = {p: d(0, p) for p in range(P)}
    tri = {p: d(7, p)[-1] for p in range(P)}
    # forward A: x block sent in place, unpacked by the library's boxes
    recv = xchg(x[:, h0:h0 + hn, w0:w0 + wn].ravel().copy(), d(1), P)
    full = np.zeros(cn * nlat * nlon)
    run_boxes(d(5), recv, full)
    full = full.reshape(cn, nlat, nlon)
    assert np.array_equal(full, x[c0:c0 + cn])
    coef = o.sht_forward(kind, nlat, nlon, lmax, mmax, full) if cn else np.zeros((0, lmax, mmax), complex)
    # forward B: triangular payloads per destination block (dist_layout.hpp payload format)
    B = d(2)
    pay = np.zeros(max(B[P:2 * P][p] + B[0:P][p] for p in range(P)) if P else 0)
    for p in range(P):
        pl0, pln, pm0, pmn = rng[p][4:8]
        ro = d(7, p)
        for f in range(cn):
            for k in range(pln):
                ms = np.arange(pm0, min(pm0 + pmn, pl0 + k + 1))
                if ms.size == 0:
                    continue
                at = B[P + p] + f * 2 * tri[p] + 2 * (ro[k] + ms - pm0)
                pay[at], pay[at + 1] = coef[f, pl0 + k, ms].real, coef[f, pl0 + k, ms].imag
    mine = xchg(pay, B, P)
    ro = d(7)
    out = np.zeros((C, ln, mn), complex)
    for c in range(C):
        for k in range(ln):
            ms = np.arange(m0, min(m0 + mn, l0 + k + 1))
            at = c * 2 * tri[q] + 2 * (ro[k] + ms - m0)
            out[c, k, ms - m0] = mine[at] + 1j * mine[at + 1]
    cg = gather(out, l0, m0, (C, lmax, mmax))
    ref = o.sht_forward(kind, nlat, nlon, lmax, mmax, x)
    e_fwd = float(np.abs(cg - ref).max() / np.abs(ref).max())
    # inverse: A^-1 (pack own block channel-major), B^-1 boxes, received in place
    send = np.zeros(C * 2 * tri[q])
    for c in range(C):
        for k in range(ln):
            ms = np.arange(m0, min(m0 + mn, l0 + k + 1))
            at = c * 2 * tri[q] + 2 * (ro[k] + ms - m0)
            send[at], send[at + 1] = out[c, k, ms - m0].real, out[c, k, ms - m0].imag
    IA = d(3)
    got = xchg(send, IA, P)
    dense = np.zeros((cn, lmax, mmax), complex)
    for p in range(P):
        pl0, pln, pm0, pmn = rng[p][4:8]
        rop = d(7, p)
        for f in range(cn):
            for k in range(pln):
                ms = np.arange(pm0, min(pm0 + pmn, pl0 + k + 1))
                at = IA[3 * P + p] + f * 2 * tri[p] + 2 * (rop[k] + ms - pm0)
                dense[f, pl0 + k, ms] = got[at] + 1j * got[at + 1]
    yfull = o.sht_inverse(kind, nlat, nlon, dense) if cn else np.zeros((0, nlat, nlon))
    IB = d(4)
    send = np.zeros(max(IB[P + p] + IB[p] for p in range(P)))
    run_boxes(d(6), yfull.ravel(), send)
    y = xchg(send, IB, P)[:C * hn * wn].reshape(C, hn, wn)
    yg = gather(y, h0, w0, (C, nlat, nlon))
    yref = o.sht_inverse(kind, nlat, nlon, ref)
    e_inv = float(np.abs(yg - yref).max() / np.abs(yref).max())
    return e_fwd, e_inv


def disco_case(nh, nw, q, ctx, ik, ih, iw, ok, oh, ow, cut, cin, cout, seed):
    P = nh * nw
    o = oracle.orc()
    oop = o.disco_assemble(ik, ih, iw, ok, oh, ow, cut)
    rp, hi = oop["row_ptr"], oop["h_in"]
    blo = [int(hi[rp[h]:rp[h + 1]].min()) for h in range(oh)]
    bn = [int(hi[rp[h]:rp[h + 1]].max()) + 1 - blo[h] for h in range(oh)]
    d = lambda what: D.describe_disco(nh, nw, q, ih, iw, oh, ow, cin, cout, blo, bn, what)  # noqa: E731
    h0, hn, w0, wn, ho0, hon, wo0, won, cz0, czn, need0, needn = d(0)
    x = oracle.random_field((cin, ih, iw), seed)
    mix = oracle.random_field((cout, cin, 9), seed + 1)
    H = d(1)
    send = np.zeros(max([H[P + p] + H[p] for p in range(P)] + [0]))
    run_boxes(d(2), x[:, h0:h0 + hn, w0:w0 + wn].ravel().copy(), send)
    recv = xchg(send, H, P)
    rows = np.zeros(czn * needn * iw)
    run_boxes(d(3), recv, rows)
    rows = rows.reshape(czn, needn, iw)
    assert np.array_equal(rows, x[cz0:cz0 + czn, need0:need0 + needn])
    xin = np.zeros((czn, ih, iw))
    xin[:, need0:need0 + needn] = rows
    part = (o.disco_apply(oop, xin, np.ascontiguousarray(mix[:, cz0:cz0 + czn]))[:, ho0:ho0 + hon]
            if czn else np.zeros((cout, hon, ow)))
    if nw > 1:
        mx = d(6)[0]
        slots = np.zeros(nw * cout * hon * mx)
        run_boxes(d(4), np.ascontiguousarray(part).ravel(), slots)
        t = torch.from_numpy(slots)
        r = torch.empty(cout * hon * mx, dtype=torch.float64)
        dist.reduce_scatter_tensor(r, t, group=ctx.pg[D.AZIMUTH])
        y = np.zeros(cout * hon * won)
        run_boxes(d(5), r.numpy(), y)
        y = y.reshape(cout, hon, won)
    else:
        y = part
    yg = gather(np.ascontiguousarray(y), ho0, wo0, (cout, oh, ow))
    ref = o.disco_apply(oop, x, mix)
    return float(np.abs(yg - ref).max() / np.abs(ref).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nh", type=int, required=True)
    ap.add_argument("--nw", type=int, required=True)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    dist.init_process_group("gloo")
    ctx = D.DistContext(D.CommGrid((1, 1, args.nh, args.nw)))
    q = dist.get_rank()
    rep = {
        "sht_ga16": sht_case(args.nh, args.nw, q, GA, 16, 32, 16, 16, 5, 30),
        "sht_eq91": sht_case(args.nh, args.nw, q, EQ, 91, 180, 91, 90, 3, 1),
        "disco_ga16": disco_case(args.nh, args.nw, q, ctx, GA, 16, 32, GA, 8, 16, 3 * PI / 8, 3, 2, 33),
        "disco_eq9": disco_case(args.nh, args.nw, q, ctx, EQ, 9, 16, EQ, 9, 16, 3 * PI / 9, 2, 1, 35),
        "disco_eq91": disco_case(args.nh, args.nw, q, ctx, EQ, 91, 180, GA, 45, 90, 3 * PI / 45, 5, 3, 37),
    }
    if q == 0:
        with open(args.out, "w") as f:
            json.dump(rep, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
