// Grouped "TN" GEMM engine shared by every contraction on the hot path:
//   D_g[M_g x N_g] = A_g[M_g x K_g] * B_g[N_g x K_g]^T        (fp32 in/out)
// Both operands are K-major (row-major with K contiguous).  A is the DATA operand
// (fields / Fourier bins), B is a constant TABLE (Legendre Phat, channel-mix weights)
// whose tf32 hi/lo split is precomputed on the host.  Groups are e.g. the (m, parity)
// blocks of the Legendre contraction (harmonics.hpp:147-154 / :184-194).
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace sph {

// Rows per field tile of the inverse SHT's EOi layout (GroupedGemm::d_mode 1):
// EOi[r][t][g][EOI_TILE], r ring pair, t = row / EOI_TILE, g = 2 m + parity.  128 rows: a
// CTA's 4 epilogue warps write each (r, t, g) run of 512 B together (32 rows measured
// 128-byte pieces 11.8 MB apart at cfg2: the inverse GEMM's epilogue cost 0.77 of 2.27 ms).
constexpr int EOI_TILE = 128;

struct GemmGroup {
    int32_t a_row0;  // first row of this group in the 2D A tensor
    int32_t b_row0;  // first row of this group in the 2D B tensor
    int32_t M, N, K;
    int32_t ldd;     // D row stride (floats)
    int32_t zero_to; // STORE_ROW: columns [N, zero_to) of each row are zero-filled
    int64_t d_off;   // element offset of D(0,0)
};

struct GemmTile {
    int32_t group, m0, n0, pad;
};

// One output tile of the tcgen05 kernel, flattened from (group, m0, n0) on the host so
// each warp role reads ONE descriptor per tile (and loads the next one a tile ahead)
// instead of two dependent global loads on the pipeline's critical path.
struct GemmWork {
    int32_t a_row;    // group a_row0 + m0
    int32_t b_row;    // group b_row0 + n0
    int32_t M;        // group rows (row validity: m < M)
    int32_t m0, n0;   // tile origin inside the group
    int32_t nrem;     // min(bn, N - n0): columns computed
    int32_t K;
    int32_t ldd;
    int32_t ncols;    // STORE_ROW columns written incl. the zero fill up to zero_to
    int32_t dg;       // group index in the 3D [group][rows][ldd] view of D (TMA store)
    int32_t ag;       // group index in the 4D quad-interleaved view of A (a_quad)
    int32_t pad;
    int64_t d_off;    // element offset of D(0,0) of the group
};

struct GemmTileList {
    DevBuf<GemmWork> d;
    int64_t n = 0;
};

enum GemmStore : int {
    STORE_ROW = 0,   // D[d_off + m*ldd + n]
    STORE_TRANS = 1, // D[d_off + n*ldd + m]
};

// 2D fp32 matrix view [rows][cols], row stride ld floats (ld*4 % 16 == 0).
struct Mat2D {
    const float* p = nullptr;
    int64_t rows = 0, cols = 0, ld = 0;
};

// A prepared grouped problem (host-side tile list + device copies).  Rebuilt when
// the group list changes; kept in plan caches.
struct GroupedGemm {
    Mat2D A, Bhi, Blo;             // Blo may be empty for SPH_PREC_TF32
    std::vector<GemmGroup> groups; // host copy
    int store = STORE_ROW;
    int bn = 256;                  // N tile (<= 256, multiple of 16)
    int cluster = 0;               // CTAs per cluster sharing the table tile (0 = auto)
    bool alo = false;              // bn 64 / 128: the BK = 32 A_lo-in-TMEM kernel (bn 192 always is)
    int ks = 1;                    // 32-wide atoms per pipeline stage (1 or 2; A_lo-in-TMEM kernels)
    bool row_tma = false;          // non-ALO STORE_ROW: TMA-store epilogue (uniform D groups)
    // blo_conv (3xTF32, bn = 192): Bhi is the RAW fp32 table and no lo table is loaded; the
    // converter warps split the SMEM tile in place (hi = rna_tf32(B), lo = B - hi, the host
    // split's values) next to A_lo: half the table's TMA bytes
    bool blo_conv = false;
    bool pair = false;             // cta_group::2 CTA-pair MMA (set by finalize)
    // TMA-store epilogue (ALO kernel): D is a uniform 3D [d_groups3][d_rows][ldd] view
    // (every group has the same ldd and row count, d_off a multiple of d_rows * ldd)
    bool tma_store = false;
    // a_quad: A is k-quad interleaved per group, element (group g, row, k) at
    // ((g * a_kq + k / 4) * a_rows_g + row) * 4 + k % 4 (the forward SHT's E/O layout,
    // fft.cu FoldIO); a_row0 of every group is g * a_rows_g.  Only with bn = 192 (ALO).
    bool a_quad = false;
    int64_t a_rows_g = 0, a_groups = 0, a_kq = 0;
    // d_mode 1 (STORE_TRANS only): D element (group dg, n, m) at
    // ((n * d_t + m / EOI_TILE) * d_g2 + dg) * EOI_TILE + m % EOI_TILE, dg = d_off / (N * ldd):
    // the inverse SHT's field-tile-major EOi, so each unfold CTA reads contiguous runs (fft.cu)
    int d_mode = 0;
    int64_t d_t = 0, d_g2 = 0;
    int64_t d_rows = 0, d_groups3 = 0, d_ldd = 0;
    DevBuf<GemmGroup> d_groups;
    int64_t ntiles = 0;            // tiles at cluster size 1 (0 -> nothing to do)
    mutable std::map<int, std::unique_ptr<GemmTileList>> tile_lists;
    std::unique_ptr<std::mutex> tiles_mu = std::make_unique<std::mutex>();
    const GemmTileList& tiles_for(int cl) const;
    DevBuf<GemmTile> d_tiles_simt;  // 64x64 tiles for the SIMT anchor
    int64_t ntiles_simt = 0;
    double flops = 0;              // algorithmic 2*M*N*K summed over groups
    const char* name = "gemm_tf32x3";  // profiler tag
    void finalize();               // build the LPT-ordered tile list, upload
};

// Run D = A*B^T for all groups with the requested precision mode
// (SPH_PREC_3XTF32 / SPH_PREC_TF32 -> tcgen05 kernel, SPH_PREC_FP32_SIMT -> SIMT).
// A.p of the prepared problem is ignored; the data operand is passed per call so a
// cached problem can serve concurrent calls on different buffers.
// Bhi/Blo override the prepared table pointers when non-null (per-call weights).
// Fused epilogue applied to the accumulator before the store (column n = output
// column, D element e): mode 1 (STORE_ROW): D = gelu_erfc(acc + bias[n]) -- the MLP's first
// layer (model.hpp:361-362); mode 2 (STORE_TRANS): D = res[e] + scale[n] * (acc + bias[n])
// -- the layer-scaled residual (model.hpp:363-368), res laid out like D.
struct GemmEpi {
    int mode = 0;
    const float* bias = nullptr;
    const float* scale = nullptr;
    const float* res = nullptr;
};

void gemm_run(const GroupedGemm& g, const float* A, float* D, int prec, cudaStream_t stream,
              const float* Bhi = nullptr, const float* Blo = nullptr, const GemmEpi* epi = nullptr);

// SMs the persistent tcgen05 GEMM may occupy for launches from this thread (0 = all).
// A scope that runs compute while NCCL kernels progress on another stream caps it, so the
// communication kernels find SMs: a persistent CTA that waits for an SM would stall its
// whole static tile stream.
struct GemmSmCap {
    int prev;
    explicit GemmSmCap(int sms);
    ~GemmSmCap();
    GemmSmCap(const GemmSmCap&) = delete;
    GemmSmCap& operator=(const GemmSmCap&) = delete;
};
int gemm_sm_cap();

// Host helpers: split fp32 table values into tf32 hi (round-to-nearest) and lo.
void tf32_split_host(const float* x, size_t n, float* hi, float* lo);

}  // namespace sph
