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

struct GemmTileList {
    DevBuf<GemmTile> d;
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
void gemm_run(const GroupedGemm& g, const float* A, float* D, int prec, cudaStream_t stream,
              const float* Bhi = nullptr, const float* Blo = nullptr);

// Host helpers: split fp32 table values into tf32 hi (round-to-nearest) and lo.
void tf32_split_host(const float* x, size_t n, float* hi, float* lo);

}  // namespace sph
