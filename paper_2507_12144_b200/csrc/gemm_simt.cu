// fp32 FMA (SIMT) grouped GEMM: the parity anchor (SPH_PREC_FP32_SIMT) behind the
// same GroupedGemm descriptor as the tcgen05 kernel.  64x64 output tile per CTA,
// 256 threads, 4x4 outputs per thread, K staged through shared memory.
#include "gemm.cuh"

namespace sph {

namespace {
constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256) gemm_simt_kernel(const float* __restrict__ A, int64_t lda,
                                                        const float* __restrict__ B,
                                                        const float* __restrict__ Blo, int64_t ldb,
                                                        const GemmGroup* __restrict__ groups,
                                                        const GemmTile* __restrict__ tiles,
                                                        float* __restrict__ D, int store,
                                                        int64_t a_rows_g, int64_t a_kq, int d_mode,
                                                        int64_t d_t, int64_t d_g2, int64_t d_gsz,
                                                        GemmEpi epi) {
    __shared__ float As[TK][TM + 4];
    __shared__ float Bs[TK][TN + 4];
    const GemmTile tl = tiles[blockIdx.x];
    const GemmGroup g = groups[tl.group];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[4][4] = {};
    const float* Ag = A + static_cast<int64_t>(g.a_row0 + tl.m0) * lda;
    const float* Bg = B + static_cast<int64_t>(g.b_row0 + tl.n0) * ldb;
    const float* Blg = Blo ? Blo + static_cast<int64_t>(g.b_row0 + tl.n0) * ldb : nullptr;
    for (int k0 = 0; k0 < g.K; k0 += TK) {
        for (int i = threadIdx.x; i < TM * TK; i += 256) {
            const int r = i / TK, kk = i % TK;
            const bool ok = (tl.m0 + r < g.M) && (k0 + kk < g.K);
            float v = 0.f;
            if (ok && a_rows_g > 0) {  // quad-interleaved A (GroupedGemm::a_quad)
                const int64_t grow = g.a_row0 + tl.m0 + r, gi = grow / a_rows_g, row = grow - gi * a_rows_g;
                const int k = k0 + kk;
                v = A[((gi * a_kq + k / 4) * a_rows_g + row) * 4 + (k & 3)];
            } else if (ok) {
                v = Ag[static_cast<int64_t>(r) * lda + k0 + kk];
            }
            As[kk][r] = v;
        }
        for (int i = threadIdx.x; i < TN * TK; i += 256) {
            const int r = i / TK, kk = i % TK;
            const bool ok = (tl.n0 + r < g.N) && (k0 + kk < g.K);
            // hi + lo reassembles the fp32 table value exactly
            const int64_t o = static_cast<int64_t>(r) * ldb + k0 + kk;
            Bs[kk][r] = ok ? (Blo ? Bg[o] + Blg[o] : Bg[o]) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* dbase = D + g.d_off;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = tl.m0 + ty * 4 + i;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = tl.n0 + tx * 4 + j;
            if (n >= g.N) continue;
            if (store == STORE_ROW) {
                float v = acc[i][j];
                if (epi.mode == 1) {
                    v += epi.bias[n];
                    v = v * 0.5f * erfcf(-v * 0.70710678118654752440f);
                }
                dbase[static_cast<int64_t>(m) * g.ldd + n] = v;
                if (n == g.N - 1)
                    for (int z = g.N; z < g.zero_to; ++z)
                        dbase[static_cast<int64_t>(m) * g.ldd + z] = 0.f;
            }
            else if (d_mode == 1)
                D[((static_cast<int64_t>(n) * d_t + m / EOI_TILE) * d_g2 + g.d_off / d_gsz) * EOI_TILE + (m % EOI_TILE)] =
                    acc[i][j];
            else if (epi.mode == 2) {
                const int64_t e = g.d_off + static_cast<int64_t>(n) * g.ldd + m;
                D[e] = epi.res[e] + epi.scale[n] * (acc[i][j] + epi.bias[n]);
            } else
                dbase[static_cast<int64_t>(n) * g.ldd + m] = acc[i][j];
        }
    }
}
}  // namespace

void build_simt_tiles(GroupedGemm& g) {
    std::vector<GemmTile> t;
    for (size_t gi = 0; gi < g.groups.size(); ++gi) {
        const GemmGroup& gr = g.groups[gi];
        if (gr.M <= 0 || gr.N <= 0 || gr.K <= 0) continue;
        for (int n0 = 0; n0 < gr.N; n0 += TN)
            for (int m0 = 0; m0 < gr.M; m0 += TM) t.push_back({static_cast<int32_t>(gi), m0, n0, 0});
    }
    g.ntiles_simt = static_cast<int64_t>(t.size());
    g.d_tiles_simt.alloc(std::max<size_t>(t.size(), 1), false);
    if (!t.empty())
        SPH_CUDA(cudaMemcpy(g.d_tiles_simt.p, t.data(), t.size() * sizeof(GemmTile),
                            cudaMemcpyHostToDevice));
}

void gemm_run_simt(const GroupedGemm& g, const float* A, const float* Bhi, const float* Blo,
                   float* D, cudaStream_t st, const GemmEpi& epi) {
    if (g.ntiles_simt == 0) return;
    ProfScope prof("gemm_simt", st, g.flops);
    gemm_simt_kernel<<<static_cast<unsigned>(g.ntiles_simt), 256, 0, st>>>(
        A, g.A.ld, Bhi, Blo, g.Bhi.ld, g.d_groups.p, g.d_tiles_simt.p, D, g.store,
        g.a_quad ? g.a_rows_g : 0, g.a_kq, g.d_mode, g.d_t, g.d_g2,
        g.d_mode == 1 ? g.d_rows * g.d_ldd : 1, epi);
    SPH_LAUNCH_CHECK();
    count_launch();
}

}  // namespace sph
