// Shared indexing of the C_int <-> order-major tile transposes (sht.cu: cint_to_dense /
// dense_to_cint; dist.cu: cint_pack / cint_unpack).
//
// C_int is [(m*2 + p)][2F (f, re/im)][Lp] with l = m + p + 2 lp.  A CTA tile covers 32
// orders x DL = 64 degrees of one field, staged in shared memory as tre/tim[64][33] with
// the degree rows split by parity (srow = (dl & 1) * 32 + dl / 2), so a warp walking one
// C_int row (every other degree) hits consecutive shared-memory rows (stride 33 words,
// conflict-free) and an order-major row is one shared-memory row.
//
// The transposes are instruction-bound (ncu at cfg2: issue slots 85-87 % busy, IPC 3.4,
// DRAM 20-36 % of peak), so the index arithmetic is strength-reduced: row r = warp + 8 i
// of a warp has a fixed parity p = (warp >> 1) & 1 and re/im ri = warp & 1 and order
// mlt = warp / 4 + 2 i (C_int row offsets advance by 4 groups = 8 F Lp floats per i); its
// 32 lanes cover degrees l = lt + off0 + 2 lane, i.e. shared-memory rows s0 + lane.
// Kernels walk their 16 rows incrementally (d -= 2, L(m, p) -= 1, row pointer += 8 F Lp):
// the multiply-per-row form left 345 IMADs in dense_to_cint, this one 154.
#pragma once

namespace sph {

template <int DL>
__device__ __forceinline__ int srow_of(int dl) {
    return (dl & 1) * (DL / 2) + (dl >> 1);
}

struct TileRow {
    int lp0, s0, off0;  // first lp of the row's run, its smem row, its degree offset in the tile
    // d = lt - m - p: the tile's first degree relative to the row's first degree
    __device__ __forceinline__ explicit TileRow(int d) {
        off0 = d > 0 ? (d & 1) : -d;
        lp0 = d > 0 ? (d + 1) >> 1 : 0;
        s0 = (off0 & 1) * 32 + (off0 >> 1);
    }
};

}  // namespace sph
