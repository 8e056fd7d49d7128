// DISCO convolution plan (convolution.hpp:141-220) + spectral convolution
// (convolution.hpp:286-304) + block epilogue (model.hpp:355-368).
#pragma once

#include <functional>
#include <vector>

#include "fft.cuh"
#include "gemm.cuh"
#include "sht.cuh"

namespace sph {

// Morlet / isotropic filter basis (convolution.hpp:30-81)
struct Basis {
    double cutoff = 0;
    std::vector<std::pair<int, int>> pairs;
    int n_real() const;
    double eval_real(int k, double theta, double phi) const;
};
Basis make_basis(int kind, double cutoff);

struct DiscoPlan {
    int device = 0;
    int in_kind = 0, out_kind = 0;
    int64_t hin = 0, win = 0, hout = 0, wout = 0;
    int K = 0;
    int64_t stride = 1, nnz = 0;
    std::vector<double> in_colat, in_w, out_colat, out_w;
    // assembled operator, reference entry order: row h holds entries
    // [row_ptr[h], row_ptr[h+1]); vals[e*K + k] = b_k * w_in (fp64 on host)
    std::vector<int64_t> row_ptr;
    std::vector<int32_t> h_in, w_rel;
    std::vector<double> vals;
    std::vector<double> bases;  // b_k without the input weight (transpose, convolution.hpp:251)
    // device: direct-gather anchor tables
    DevBuf<int64_t> d_row_ptr;
    DevBuf<int32_t> d_h_in, d_w_rel;
    DevBuf<float> d_vals;
    // device: longitude-Fourier tables.  band of input rows per output row,
    // psi_hat[(psi_off[h] + bi) * nbi + m][k] complex = sum_e psi_k[e] e^{-2 pi i w_rel m / win}
    std::vector<int32_t> band0, bandc;
    std::vector<int64_t> psi_off;
    DevBuf<int32_t> d_band0, d_bandc;
    DevBuf<int64_t> d_psi_off;
    DevBuf<float2> d_psi_hat;
    int64_t nbi = 0, nbo = 0;  // win/2+1, wout/2+1
    FftPlan fft_in, fft_out;
    int prec = SPH_PREC_3XTF32;

    // transpose (disco_transpose_apply, convolution.hpp:226-266), built on first use:
    // psi_t_hat[(psi_off[h] + bi) * nbi + m][k] = sum_e b_k w_out[h] e^{-2 pi i w_rel m / win}
    // and the row-tile map: input rows [16 t, 16 t + 16) are touched by the output rows
    // tb_h[tb_ptr[t] .. tb_ptr[t+1]) (those whose band meets the tile)
    bool t_ready = false;
    DevBuf<float2> d_psi_t;
    DevBuf<int32_t> d_tb_ptr, d_tb_h;
    int64_t t_max_pairs = 0, t_max_h = 0;  // per row tile: (h, r) band pairs, output rows
    void build_transpose();

    std::mutex mu;
    std::map<std::tuple<int64_t, int64_t, int64_t, int64_t>, std::unique_ptr<GroupedGemm>> gemm_cache;
    // k-split of the 3xTF32 mix reduction (c_in * K > kchunk): chunk GEMMs keyed by
    // (B, cin, cout, nout, k0, kc), each writing its own partial spectrum
    std::map<std::tuple<int64_t, int64_t, int64_t, int64_t, int64_t, int64_t>, std::unique_ptr<GroupedGemm>>
        gemm_chunk_cache;
    std::map<std::tuple<int64_t, int64_t, int64_t>, std::unique_ptr<GroupedGemm>> gemm_t_cache;
    DevBuf<uint8_t> own_ws;

    void create(int in_kind, int64_t in_nlat, int64_t in_nlon, int out_kind, int64_t out_nlat,
                int64_t out_nlon, int basis, double cutoff, int flags);
    int64_t workspace_bytes(int64_t B, int64_t cin, int64_t cout) const;
    void apply(const float* x, const float* mix, int64_t B, int64_t cin, int64_t cout, float* y,
               void* ws, cudaStream_t st);
    // output rows [ho0, ho0+nout) from input rows [h_in0, h_in0+nin) (latitude shards)
    // make_u (optional): produces the channel-minor input spectrum U[B][nin][nbi][cin]
    // instead of the R2C of x (the fused decoder builds it from the latent's spectrum)
    void apply_rows(const float* x, int64_t h_in0, int64_t nin, int64_t ho0, int64_t nout,
                    const float* mix, int64_t B, int64_t cin, int64_t cout, float* y, void* ws,
                    cudaStream_t st, const std::function<void(float2*)>* make_u = nullptr);
    // U layout of the band stage: channel pairs interleaved (FFMA2 band kernel) for even cin
    bool pair_layout(int64_t cin) const;
    void input_rows(int64_t ho0, int64_t nout, int64_t* lo, int64_t* n) const;
    int64_t rows_workspace_bytes(int64_t B, int64_t cin, int64_t cout, int64_t nin, int64_t nout) const;
    // v [B][cout][hout][wout] on the output grid -> y [B][cin][hin][win] on the input grid
    void transpose_apply(const float* v, const float* mix, int64_t B, int64_t cin, int64_t cout,
                         float* y, void* ws, cudaStream_t st);
    int64_t transpose_workspace_bytes(int64_t B, int64_t cin, int64_t cout) const;
};

void spectral_conv(ShtPlan& p, const float* x, const float* kernel, int64_t B, int64_t cin,
                   int64_t cout, int64_t klmax, float* y, void* ws, cudaStream_t st);
int64_t spectral_conv_ws_bytes(const ShtPlan& p, int64_t B, int64_t cin, int64_t cout);
// the mix stage alone on reference-layout coefficients [B][cin][lmax][mmax] complex64 ->
// [B][cout][lmax][mmax] (same workspace size as spectral_conv)
void spectral_mix(ShtPlan& p, const float* coeffs, const float* kernel, int64_t B, int64_t cin, int64_t cout,
                  int64_t klmax, float* out, void* ws, cudaStream_t st);

void block_epilogue(const float* conv, const float* x, const float* w1, const float* b1,
                    const float* w2, const float* b2, const float* scales, int64_t B, int64_t C,
                    int64_t H, int64_t npts, float* y, cudaStream_t st);

// fp32 -> tf32 hi/lo split of a device matrix [rows][cols] into [rows][ld] (zero padded)
void split_rows(const float* src, int64_t rows, int64_t cols, int64_t ld, float* hi, float* lo,
                cudaStream_t st);

}  // namespace sph
