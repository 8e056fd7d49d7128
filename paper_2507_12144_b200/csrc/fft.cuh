// Longitude ring transforms (fft.hpp:97-113 rfft_bins / real_synthesis) for sm_100a.
//
// Two real rings are packed into one complex ring z = a + i b and transformed in
// shared memory (register four-step for n = N1*45, mixed-radix Stockham otherwise).  The forward epilogue splits
// A = (Z + conj Z_{N-k})/2, B = (Z - conj Z_{N-k})/2i and writes the parity-folded
// E = A + B / O = A - B straight into the Legendre GEMM operand layout; the inverse
// prologue builds Z from Ev +- Od (harmonics.hpp:188-193 Hermitian completion).
#pragma once

#include <vector>

#include "common.cuh"

namespace sph {

constexpr int FFT_THREADS = 256;
constexpr int FFT_MAX_STAGES = 24;

struct FftPlan {
    int n = 0;
    int nstages = 0;
    int radix[FFT_MAX_STAGES] = {};
    bool direct = false;     // n has a prime factor > 5: O(n^2) fallback kernel
    DevBuf<float2> tw;       // W_n^q = exp(-2 pi i q / n), q = 0..n-1 (fp64 -> fp32)
    int rows_per_block = 1;  // rings (complex) per CTA of the Stockham engine
    int fft4_n1 = 0;         // n = fft4_n1 * 45 -> register four-step engine (fft4.cuh)
    DevBuf<float2> twT;      // four-step inter-twiddles W_n^{n2 k1} at [k1*45 + n2]
    void build(int n_);
};

// Folded-row description shared with the SHT plan: row r of the folded problem
// pairs latitude ia[r] with its mirror ib[r] (theta_b = pi - theta_a), ib = -1 if
// the row is its own mirror (pole row of the reference equiangular grid, equator).
struct FoldRows {
    int R = 0;
    std::vector<int2> rows;  // (ia, ib)
    DevBuf<int2> d_rows;
};

// Optional ring addressing for the SHT ring transforms: ring (field f, latitude row h) at
// base + f * fstr[h] + roff[h] (device arrays over latitude rows) instead of the dense
// [F][nlat][nlon] layout -- the distributed SHT reads / writes its all-to-all stage buffers
// in place (csrc/dist.cu).  Null pointers: the dense layout.
struct RingRows {
    const int64_t* roff = nullptr;
    const int64_t* fstr = nullptr;
};

// Forward: x [F][nlat][nlon] -> EO[(m*2+p)*2F + 2f+reim][r] (row stride ld_eo),
// m < mmax.  (E for p = 0, O for p = 1; raw DFT sums, no 2pi/nlon scale.)
void fft_forward_fold(const FftPlan& fp, const FoldRows& fr, const float* x, int64_t F,
                      int nlat, int mmax, float* eo, int64_t ld_eo, cudaStream_t st, RingRows rr = {});

// Inverse: EOi[(m*2+p)][r][2f+reim] (Ev/Od per folded row, the inverse GEMM's
// transposed store; ld_eo unused) -> y [F][nlat][nlon].
// Orders m < msynth are used; groups (m,p) with no Legendre degrees (L_mp = 0) are
// treated as zero: L_mp = number of l in [m, lmax) with (l - m) % 2 == p.
void fft_inverse_unfold(const FftPlan& fp, const FoldRows& fr, const float* eoi, int64_t F,
                        int nlat, int mmax, int msynth, int lmax, int64_t ld_eo, float* y,
                        cudaStream_t st, RingRows rr = {});

// Plain forward ring transform for the distributed stage (distsim.hpp:413-430):
// rings [nrings][nlon] -> bins [nrings][nbins] complex64, scaled by `scale`.
void fft_forward_plain(const FftPlan& fp, const float* rings, int64_t nrings, int nbins,
                       float scale, float2* bins, cudaStream_t st);

// Plain C2R: bins [nrings][nbins] complex half spectra (bins >= nbins are zero,
// Im of DC / Nyquist ignored) -> rings [nrings][n] real, times `scale`.  nparts > 1: the
// spectrum is the fp32 sum of nparts partial spectra part_stride float2 apart (the DISCO
// mix's k-split partials), added while loading.
void fft_inverse_plain(const FftPlan& fp, const float2* bins, int64_t nrings, int nbins,
                       float scale, float* rings, cudaStream_t st, int nparts = 1, int64_t part_stride = 0);

// Channel-minor forward transform for DISCO: x [B][C][H][n] ->
// U [B][H][nbins][C] complex (bins m < nbins, unscaled).  planar = 1: real planes
// [(b, h, m, re/im)][ldp]; planar = 2: channel pairs interleaved (re c, re c+1, im c, im c+1).
void fft_forward_cminor(const FftPlan& fp, const float* x, int64_t B, int64_t C, int64_t H,
                        int nbins, float2* U, cudaStream_t st, int planar = 0, int64_t ldp = 0);
// channel-minor C2R: half spectra V[B][H][nbins][C] -> rings y[B][C][H][n] * scale
void fft_inverse_cminor(const FftPlan& fp, const float2* V, int64_t B, int64_t C, int64_t H, int nbins,
                        float scale, float* y, cudaStream_t st);

}  // namespace sph
