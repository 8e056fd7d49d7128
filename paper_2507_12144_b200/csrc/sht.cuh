// SHT plan: host fp64 precompute + device tables + orchestration of
//   forward  x --fft_forward_fold--> EO --grouped GEMM (Pf)--> C_int
//   inverse  C_int --grouped GEMM (Pi)--> EO_i --fft_inverse_unfold--> y
// (harmonics.hpp:126-205, distsim.hpp:404-463).
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "fft.cuh"
#include "gemm.cuh"

namespace sph {

// grid.hpp:69-128 restated in the product (fp64, host)
void build_grid(int kind, int64_t nlat, int64_t nlon, std::vector<double>& colat,
                std::vector<double>& w);

struct ShtPlan {
    int device = 0;
    int kind = 0;
    int64_t nlat = 0, nlon = 0, lmax = 0, mmax = 0;
    int flags = 0, prec = SPH_PREC_3XTF32;
    int64_t msynth = 0;
    std::vector<double> colat, w;
    FoldRows fold;
    int R = 0, Rp = 0;        // folded rows, padded row stride of EO / Pf
    int Lmax_p = 0, Lp = 0;   // max degrees per parity class, padded stride of C_int / Pi
    FftPlan fft;
    // Pf: [(m,p) blocks of L_mp rows][Rp]  (Phat * quadrature weight)
    DevBuf<float> pf_hi, pf_lo;
    std::vector<int64_t> pf_off;  // first row of block (m,p), size 2*mmax
    int64_t pf_rows = 0;
    // Pi: [(m,p)][R][Lp]  (Phat)
    DevBuf<float> pi_hi, pi_lo;

    std::mutex mu;
    std::map<int64_t, std::unique_ptr<GroupedGemm>> fwd_cache, inv_cache;
    std::map<std::tuple<int64_t, int64_t, int64_t>, std::unique_ptr<GroupedGemm>> stage_cache;
    DevBuf<uint8_t> own_ws;

    int64_t L(int64_t m, int p) const {  // degrees l in [m, lmax) with (l-m)%2 == p
        const int64_t n = lmax - m;
        return n <= 0 ? 0 : (p == 0 ? (n + 1) / 2 : n / 2);
    }
    // E/O (forward, quad-interleaved) and EOi (inverse, field tiles of 32 rows) share it
    int64_t eo_elems(int64_t F) const { return mmax * 2 * ((2 * F + EOI_TILE - 1) / EOI_TILE * EOI_TILE) * Rp; }
    int64_t cint_elems(int64_t F) const { return mmax * 2 * 2 * F * Lp; }
    int64_t dense_elems(int64_t F) const { return F * lmax * mmax * 2; }
    int64_t workspace_bytes(int64_t F) const { return 4 * (eo_elems(F) + cint_elems(F)) + 256; }

    void create(int kind, int64_t nlat, int64_t nlon, int64_t lmax, int64_t mmax, int flags);
    const GroupedGemm& fwd_gemm(int64_t F);
    const GroupedGemm& inv_gemm(int64_t F);
    const GroupedGemm& stage_gemm(int64_t F, int64_t m0, int64_t mcount);
    void* workspace(void* ws, int64_t bytes);

    // rr: optional ring addressing of x / y (fft.cuh RingRows; the distributed SHT's stage
    // buffers), default the dense [F][nlat][nlon] layout
    void forward(const float* x, int64_t F, float* out, int layout, void* ws, cudaStream_t st,
                 RingRows rr = {});
    void inverse(const float* coeffs, int64_t F, int layout, float* y, void* ws, cudaStream_t st,
                 RingRows rr = {});
    void fft_stage(const float* rings, int64_t F, int64_t h, float* bins, cudaStream_t st);
    void legendre_stage(const float* bins, int64_t F, int64_t m0, int64_t mcount, float* coeffs,
                        void* ws, cudaStream_t st);
    int64_t stage_ws_bytes(int64_t F, int64_t mcount) const {
        return 4 * (mcount * 2 * 2 * F * (int64_t)Rp + mcount * 2 * 2 * F * (int64_t)Lp) + 256;
    }
    // host round trip: pinned host x -> (H2D | SHT+ISHT | D2H) pipeline -> host y
    void roundtrip_host(const float* xh, int64_t F, float* yh, int64_t chunk);
    struct HostPipe;
    std::unique_ptr<HostPipe> pipe;  // cached streams / events / chunk buffers
    std::mutex pipe_mu;
    ShtPlan();
    ~ShtPlan();
};

// C_int <-> reference dense [F][lmax][mmax] complex64 conversions
void cint_to_dense(const ShtPlan& p, const float* cint, int64_t F, int64_t m0, int64_t mcount,
                   int64_t out_mcount, float* dense, cudaStream_t st);
void dense_to_cint(const ShtPlan& p, const float* dense, int64_t F, float* cint, cudaStream_t st);

}  // namespace sph
