// Spherical harmonic transforms on sm_100a (see sht.cuh).
//
// Parity folding.  The reference grids are symmetric about the equator: Gaussian
// nodes pair i <-> nlat-1-i, the reference equiangular grid pairs i <-> nlat-i (its
// pole row theta = 0 has no mirror, grid.hpp:80-83).  With x_b = -x_a and
// Phat_l^m(-x) = (-1)^(l+m) Phat_l^m(x), the contraction over latitude
// (harmonics.hpp:147-154) splits per order m into two half-size contractions:
//   uhat_lm = sum_r Pw_lm(x_r) E_r   (l-m even),   sum_r Pw_lm(x_r) O_r  (l-m odd)
// with E_r = G_a + G_b, O_r = G_a - G_b, and the synthesis (harmonics.hpp:184-187)
// returns Ev+Od on ring a and Ev-Od on ring b.  Unpaired rows enter both classes
// with G_b = 0.  Each (m, parity) block is one group of the grouped GEMM.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <thread>

#include "sht.cuh"
#include "tile_rows.cuh"

namespace sph {

void build_grid(int kind, int64_t nlat, int64_t nlon, std::vector<double>& colat,
                std::vector<double>& w) {
    const double pi = 3.14159265358979323846;
    if (kind == SPH_EQUIANGULAR) {
        require(nlat >= 2 && nlon >= 2, "build_equiangular: nlat and nlon must be >= 2");
        colat.resize(nlat);
        w.resize(nlat);
        const double wfac = 2.0 * pi * pi / (static_cast<double>(nlat) * static_cast<double>(nlon));
        for (int64_t i = 0; i < nlat; ++i) {
            colat[i] = pi * static_cast<double>(i) / static_cast<double>(nlat);
            w[i] = wfac * std::sin(colat[i]);
        }
        return;
    }
    require(kind == SPH_GAUSSIAN, "grid: unknown grid kind");
    require(nlat >= 1 && nlon >= 2, "build_gaussian: need nlat >= 1 and nlon >= 2");
    colat.resize(nlat);
    w.resize(nlat);
    const double dphi = 2.0 * pi / static_cast<double>(nlon);
    auto pn_dpn = [](int64_t n, double x, double& pn, double& dpn) {
        double p0 = 1.0, p1 = x;
        if (n == 0) { pn = 1.0; dpn = 0.0; return; }
        for (int64_t k = 2; k <= n; ++k) {
            const double kk = static_cast<double>(k);
            const double p2 = ((2.0 * kk - 1.0) * x * p1 - (kk - 1.0) * p0) / kk;
            p0 = p1;
            p1 = p2;
        }
        pn = p1;
        dpn = static_cast<double>(n) * (x * p1 - p0) / (x * x - 1.0);
    };
    for (int64_t i = 0; i < nlat; ++i) {
        double x = std::cos(pi * (static_cast<double>(i) + 0.75) / (static_cast<double>(nlat) + 0.5));
        double pn = 0, dpn = 0;
        bool ok = false;
        for (int it = 0; it < 100; ++it) {
            pn_dpn(nlat, x, pn, dpn);
            const double dx = pn / dpn;
            x -= dx;
            if (std::abs(dx) <= 1e-15) { ok = true; break; }
        }
        if (!ok) fail(SPH_ERR_RUNTIME, "build_gaussian: Newton iteration failed at node " + std::to_string(i));
        pn_dpn(nlat, x, pn, dpn);
        colat[i] = std::acos(x);
        w[i] = 2.0 / ((1.0 - x * x) * dpn * dpn) * dphi;
    }
}

namespace {

bool fwd_blo_conv() {
    static const bool on = std::getenv("SPH_GEMM_BLO_CONV_FWD") && std::atoi(std::getenv("SPH_GEMM_BLO_CONV_FWD")) != 0;
    return on;
}
bool inv_blo_conv() {
    static const bool on = !std::getenv("SPH_GEMM_BLO_CONV") || std::atoi(std::getenv("SPH_GEMM_BLO_CONV")) != 0;
    return on;
}

// Phat_l^m(x) for l in [m, lmax) by the reference recurrence (harmonics.hpp:68-100),
// fp64.  fl[l] = sqrt((4l^2-1)/(l^2-m^2)) precomputed per m.
void legendre_column(double x, int64_t m, int64_t lmax, const double* fl, double* out) {
    const double four_pi = 4.0 * 3.14159265358979323846;
    const double omx2 = (1.0 - x) * (1.0 + x);
    double pmm = 1.0, fact = 1.0;
    for (int64_t k = 1; k <= m; ++k) {
        pmm *= omx2 * fact / (fact + 1.0);
        fact += 2.0;
    }
    pmm = std::sqrt((2.0 * static_cast<double>(m) + 1.0) * pmm / four_pi);
    if (m & 1) pmm = -pmm;
    if (m < lmax) out[m] = pmm;
    if (m + 1 < lmax) {
        const double s3 = std::sqrt(2.0 * static_cast<double>(m) + 3.0);
        const double pmmp1 = x * s3 * pmm;
        out[m + 1] = pmmp1;
        double oldfact = s3, pa = pmm, pb = pmmp1;
        for (int64_t l = m + 2; l < lmax; ++l) {
            const double f = fl[l];
            const double pl = (x * pb - pa / oldfact) * f;
            out[l] = pl;
            oldfact = f;
            pa = pb;
            pb = pl;
        }
    }
}

template <class Fn>
void parallel_for(int64_t n, Fn fn) {
    int nt = static_cast<int>(std::min<int64_t>(n, std::max(1u, std::thread::hardware_concurrency())));
    nt = std::min(nt, 32);
    if (nt <= 1) {
        for (int64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int64_t i = t; i < n; i += nt) fn(i);
        });
    for (auto& t : th) t.join();
}

template <class T>
void upload(DevBuf<T>& d, const std::vector<T>& h) {
    d.alloc(h.size(), false);
    if (!h.empty()) SPH_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

// ---------------------------------------------------------------- kernels
// Internal coefficient layout <-> dense [F][lmax][mcols] complex (m contiguous): tiled
// transposes through shared memory (tile_rows.cuh), both global sides in contiguous runs.
// CTA (32 orders, 64 degrees, FPC fields): 128 cint rows (order, parity, re/im) read as
// 32-lane runs of lp (each run is the tile's 32 degrees of that parity class), dense rows
// written as 32-order float2 runs (zeros above the diagonal, decided at the store).  The
// FPC fields of a CTA share every index computation (the kernels are issue-bound).
template <int FPC>
__global__ void __launch_bounds__(256, FPC == 2 ? 3 : 4) cint_to_dense_kernel(const float* __restrict__ cint, int64_t F, int lmax,
                                                            int m0, int mcount, int out_mcount, int Lp,
                                                            float2* __restrict__ dense, int64_t f0) {
    constexpr int DL = 64, RPW = 128 / 8;
    __shared__ float tre[FPC][DL][33], tim[FPC][DL][33];
    // fields slowest: concurrently running CTAs share a field's dense rows (fields fastest,
    // for adjacent C_int rows instead, measured 2.42 vs 2.27 ms at 1024 fields)
    const int mt = blockIdx.x * 32, lt = blockIdx.y * DL;
    const int64_t f = f0 + static_cast<int64_t>(blockIdx.z) * FPC;
    const int nf = static_cast<int>(min(static_cast<int64_t>(FPC), F - f));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (m0 + mt <= lt + DL - 1) {  // else the whole tile is above the diagonal (m > l)
        const int p = (warp >> 1) & 1, ri = warp & 1;
        const int64_t gstep = 8 * F * Lp;  // 4 groups (m += 2)
        const int ml0 = mt + (warp >> 2);
        const float* rp = cint + ((static_cast<int64_t>(ml0) * 2 + p) * 2 * F + 2 * f + ri) * Lp + lane;
        float v[FPC][RPW];
        int sr[RPW];
        int d = lt - (m0 + ml0) - p;  // the row's first tile degree offset (TileRow), -2 per row
#pragma unroll
        for (int i = 0; i < RPW; ++i, d -= 2, rp += gstep) {  // all loads before any shared store
            const TileRow tr(d);
            const int lp = tr.lp0 + lane, dl = tr.off0 + 2 * lane;
            const bool ok = ml0 + 2 * i < mcount && dl < DL && lp < Lp && lt + dl < lmax;
#pragma unroll
            for (int q = 0; q < FPC; ++q) v[q][i] = ok && q < nf ? __ldg(rp + tr.lp0 + q * 2 * Lp) : 0.f;
            sr[i] = ok ? tr.s0 + lane : -1;
        }
#pragma unroll
        for (int q = 0; q < FPC; ++q) {
            float (*T)[33] = ri ? tim[q] : tre[q];
#pragma unroll
            for (int i = 0; i < RPW; ++i)
                if (sr[i] >= 0) T[sr[i]][(warp >> 2) + 2 * i] = v[q][i];
        }
    }
    __syncthreads();
    const int oc = mt + lane;
    const bool mok = oc < out_mcount;
    const bool have = mt + lane < mcount;  // orders beyond mcount are zero columns
    if (!mok) return;
    float2* dst = dense + (f * lmax + lt + warp) * out_mcount + oc;
    const int64_t dstep = 8 * static_cast<int64_t>(out_mcount), fstep = static_cast<int64_t>(lmax) * out_mcount;
    const int mabs = have ? m0 + mt + lane : lmax;  // stored entries: l >= mabs
    const int s0 = (warp & 1) * (DL / 2) + (warp >> 1);
#pragma unroll
    for (int i = 0; i < DL / 8; ++i, dst += dstep) {
        const int l = lt + warp + 8 * i;
        if (l >= lmax) break;
        const bool val = mabs <= l;
#pragma unroll
        for (int q = 0; q < FPC; ++q)
            if (q < nf)
                dst[q * fstep] = val ? make_float2(tre[q][s0 + 4 * i][lane], tim[q][s0 + 4 * i][lane])
                                     : make_float2(0.f, 0.f);
    }
}

// CTA (32 orders, 64 degrees, FPC fields): the dense rows of the tile loaded once as
// 32-order runs (no overlap between tiles); each (order, parity, re/im) C_int row gets
// the 32 consecutive lp whose degrees fall in the tile, written as one 32-lane run.  The
// degree tiles run past lmax far enough to zero every lp the inverse GEMM reads: up to
// L(m, p) rounded to its 32-wide k-block (the padding beyond that is never touched).
template <int FPC>
__global__ void __launch_bounds__(256) dense_to_cint_kernel(const float2* __restrict__ dense, int64_t F, int64_t lmax,
                                                            int64_t mmax, int Lp, float* __restrict__ cint,
                                                            int64_t f0) {
    constexpr int DL = 64, RPW = 128 / 8, EPT = DL * 32 / 256;
    __shared__ float tre[FPC][DL][33], tim[FPC][DL][33];
    const int mt = blockIdx.x * 32, lt = blockIdx.y * DL;  // fields slowest (3.60 vs 2.90 ms fastest)
    const int64_t f = f0 + static_cast<int64_t>(blockIdx.z) * FPC;
    const int nf = static_cast<int>(min(static_cast<int64_t>(FPC), F - f));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lmx = static_cast<int>(lmax), mmx = static_cast<int>(mmax);
    {  // element i: degree lt + warp + 8 i, order mt + lane; all loads before the stores
        const int m = mt + lane;
        const float2* src = dense + (f * lmax + lt + warp) * mmax + m;
        const int64_t sstep = 8 * mmax, fstep = lmax * mmax;
        const int lmin = m < mmx ? m : lmx;  // stored entries: m <= l < lmax
        float2 v[FPC][EPT];
#pragma unroll
        for (int i = 0; i < EPT; ++i, src += sstep) {
            const int l = lt + warp + 8 * i;
            const bool ok = l < lmx && lmin <= l;
#pragma unroll
            for (int q = 0; q < FPC; ++q) v[q][i] = ok && q < nf ? __ldg(src + q * fstep) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < FPC; ++q)
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int sr = (warp & 1) * (DL / 2) + (warp >> 1) + 4 * i;
                tre[q][sr][lane] = v[q][i].x;
                tim[q][sr][lane] = v[q][i].y;
            }
    }
    __syncthreads();
    const int p = (warp >> 1) & 1, ri = warp & 1;
    const int64_t gstep = 8 * F * Lp;  // 4 groups (m += 2)
    const int mw = mt + (warp >> 2);
    float* rp = cint + ((static_cast<int64_t>(mw) * 2 + p) * 2 * F + 2 * f + ri) * Lp + lane;
    int d = lt - mw - p;              // TileRow offset, -2 per row
    int lmp = (lmx - mw + 1 - p) >> 1;  // L(m, p) while m < lmax (<= 0 after), -1 per row
#pragma unroll
    for (int i = 0; i < RPW; ++i, d -= 2, --lmp, rp += gstep) {
        if (mw + 2 * i >= mmx) break;
        const TileRow tr(d);
        const int lp = tr.lp0 + lane, dl = tr.off0 + 2 * lane;
        const int lim = min(Lp, (max(lmp, 0) + 31) & ~31);
        if (dl < DL && lp < lim) {
            const bool in = lt + dl < lmx;
#pragma unroll
            for (int q = 0; q < FPC; ++q)
                if (q < nf) rp[tr.lp0 + q * 2 * Lp] = in ? (ri ? tim : tre)[q][tr.s0 + lane][(warp >> 2) + 2 * i] : 0.f;
        }
    }
}

// fields per CTA of the C_int <-> dense transposes (SPH_TR_FIELDS = 1 or 2 overrides):
// from_dense 1.76 -> 1.22 ms at cfg2 with 2; to_dense 1.40 -> 1.31-1.36 ms with 2 once its
// registers are capped for 3 CTAs/SM (uncapped: 90 registers, 2 CTAs/SM, 1.58 ms;
// profiles/r2/tr_fields_ab.log, tr_fields_ab2.log)
int tr_fields(int dflt) {
    static const int v = std::getenv("SPH_TR_FIELDS") ? std::atoi(std::getenv("SPH_TR_FIELDS")) : 0;
    return v == 1 || v == 2 ? v : dflt;
}

// bins [F][nlat][mcount] complex (scaled by 2pi/nlon) -> EO_loc [mcount][2][Rp/4][2F][4]
__global__ void fold_bins_kernel(const float2* __restrict__ bins, const int2* __restrict__ rows,
                                 int R, int Rp, int64_t F, int64_t nlat, int64_t mcount,
                                 float unscale, float* __restrict__ eo) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t twoF = 2 * F;
    if (i >= mcount * 2 * twoF * Rp) return;
    const int r = static_cast<int>(i % Rp);
    const int64_t n = (i / Rp) % twoF;
    const int64_t g = i / (static_cast<int64_t>(Rp) * twoF);
    float* dst = eo + ((g * (Rp / 4) + r / 4) * twoF + n) * 4 + (r & 3);  // quad-interleaved
    if (r >= R) {
        *dst = 0.f;
        return;
    }
    const int64_t ml = g >> 1;
    const int p = static_cast<int>(g & 1);
    const int64_t f = n >> 1;
    const int2 rw = rows[r];
    const float2 a = bins[(f * nlat + rw.x) * mcount + ml];
    const float2 b = rw.y >= 0 ? bins[(f * nlat + rw.y) * mcount + ml] : make_float2(0.f, 0.f);
    const float va = (n & 1) ? a.y : a.x, vb = (n & 1) ? b.y : b.x;
    *dst = (p == 0 ? va + vb : va - vb) * unscale;
}

}  // namespace

void cint_to_dense(const ShtPlan& p, const float* cint, int64_t F, int64_t m0, int64_t mcount,
                   int64_t out_mcount, float* dense, cudaStream_t st) {
    if (F * p.lmax * out_mcount == 0) return;
    double pairs = 0;  // stored (l, m) entries read from cint
    for (int64_t ml = 0; ml < mcount; ++ml) pairs += static_cast<double>(std::max<int64_t>(0, p.lmax - (m0 + ml)));
    ProfScope prof("sht_to_dense", st, 8.0 * F * p.lmax * out_mcount + 8.0 * F * pairs);
    const int fpc = tr_fields(2);
    for (int64_t f0 = 0; f0 < F; f0 += 65535LL * fpc) {
        const int64_t nfc = std::min<int64_t>(65535LL * fpc, F - f0);
        dim3 grid(static_cast<unsigned>((out_mcount + 31) / 32), static_cast<unsigned>((p.lmax + 63) / 64),
                  static_cast<unsigned>((nfc + fpc - 1) / fpc));
        auto k = fpc == 2 ? cint_to_dense_kernel<2> : cint_to_dense_kernel<1>;
        k<<<grid, 256, 0, st>>>(cint, F, static_cast<int>(p.lmax), static_cast<int>(m0), static_cast<int>(mcount),
                                static_cast<int>(out_mcount), p.Lp, reinterpret_cast<float2*>(dense), f0);
        SPH_LAUNCH_CHECK();
        count_launch();
    }
}

void dense_to_cint(const ShtPlan& p, const float* dense, int64_t F, float* cint, cudaStream_t st) {
    if (p.mmax * F * p.Lp == 0) return;
    ProfScope prof("sht_from_dense", st, 8.0 * F * p.lmax * p.mmax + 8.0 * F * p.lmax * (p.lmax + 1) / 2.0);
    // degree tiles up to the last zero-padded lp: l = m + p + 2 (round_up(L(m, p), 32) - 1)
    // <= m + 2 L(m, p) + 61 <= lmax + 62
    const int64_t lend = p.lmax + 63;
    const int fpc = tr_fields(2);
    for (int64_t f0 = 0; f0 < F; f0 += 65535LL * fpc) {
        const int64_t nfc = std::min<int64_t>(65535LL * fpc, F - f0);
        dim3 grid(static_cast<unsigned>((p.mmax + 31) / 32), static_cast<unsigned>((lend + 63) / 64),
                  static_cast<unsigned>((nfc + fpc - 1) / fpc));
        auto k = fpc == 2 ? dense_to_cint_kernel<2> : dense_to_cint_kernel<1>;
        k<<<grid, 256, 0, st>>>(reinterpret_cast<const float2*>(dense), F, p.lmax, p.mmax, p.Lp, cint, f0);
        SPH_LAUNCH_CHECK();
        count_launch();
    }
}

void ShtPlan::create(int kind_, int64_t nlat_, int64_t nlon_, int64_t lmax_, int64_t mmax_,
                     int flags_) {
    SPH_CUDA(cudaGetDevice(&device));
    kind = kind_;
    nlat = nlat_;
    nlon = nlon_;
    lmax = lmax_;
    mmax = mmax_;
    flags = flags_;
    prec = flags & SPH_FLAG_PREC_MASK;
    const bool adjoint = (flags & SPH_FLAG_ADJOINT) != 0;
    require(prec <= SPH_PREC_FP32_SIMT, "sht plan: unknown precision mode");
    require(lmax >= 1 && mmax >= 1, "sht plan: lmax and mmax must be >= 1");
    require(mmax <= lmax, "SpectralCoeffs: mmax must be <= lmax");
    require(nlat <= 65535 && nlon <= 65535 && lmax <= 16384, "sht plan: size out of range");
    build_grid(kind, nlat, nlon, colat, w);
    msynth = std::min<int64_t>(mmax, (nlon - 1) / 2 + 1);  // harmonics.hpp:179

    // ---- fold rows
    const double pi = 3.14159265358979323846;
    std::vector<bool> used(nlat, false);
    fold.rows.clear();
    for (int64_t i = 0; i < nlat; ++i) {
        if (used[i]) continue;
        used[i] = true;
        const double target = pi - colat[i];
        auto it = std::lower_bound(colat.begin(), colat.end(), target - 1e-9);
        int64_t j = -1;
        for (; it != colat.end() && *it <= target + 1e-9; ++it) {
            const int64_t c = it - colat.begin();
            if (c != i && !used[c]) { j = c; break; }
        }
        if (j >= 0) used[j] = true;
        fold.rows.push_back(make_int2(static_cast<int>(i), static_cast<int>(j)));
    }
    R = fold.R = static_cast<int>(fold.rows.size());
    Rp = static_cast<int>(round_up(R, 4));
    upload(fold.d_rows, fold.rows);
    Lmax_p = static_cast<int>(L(0, 0));
    Lp = static_cast<int>(round_up(Lmax_p, 4));
    fft.build(static_cast<int>(nlon));

    // ---- Legendre tables (host fp64 -> fp32 hi/lo)
    pf_off.assign(2 * mmax + 1, 0);
    for (int64_t m = 0; m < mmax; ++m)
        for (int p = 0; p < 2; ++p) pf_off[m * 2 + p + 1] = pf_off[m * 2 + p] + L(m, p);
    pf_rows = pf_off[2 * mmax];
    std::vector<float> pf(static_cast<size_t>(pf_rows) * Rp, 0.f);
    std::vector<float> pit(static_cast<size_t>(mmax) * 2 * R * Lp, 0.f);
    parallel_for(mmax, [&](int64_t m) {
        std::vector<double> fl(lmax, 0.0), col(lmax, 0.0);
        for (int64_t l = m + 2; l < lmax; ++l) {
            const double ld = static_cast<double>(l), md = static_cast<double>(m);
            fl[l] = std::sqrt((4.0 * ld * ld - 1.0) / (ld * ld - md * md));
        }
        for (int r = 0; r < R; ++r) {
            const int ia = fold.rows[r].x;
            const double x = std::cos(colat[ia]);
            legendre_column(x, m, lmax, fl.data(), col.data());
            for (int p = 0; p < 2; ++p) {
                const int64_t Lmp = L(m, p);
                for (int64_t lp = 0; lp < Lmp; ++lp) {
                    const double v = col[m + p + 2 * lp];
                    if (adjoint) {
                        // analysis A: c = sum_ij w_i P x e^{-im phi}; synthesis S doubles m >= 1
                        // (Hermitian C2R).  Under <c, d> = sum Re(conj(c) d) over stored m >= 0:
                        //   S^T z = unweighted analysis of z, m >= 1 doubled   ("forward" tables)
                        //   A^T d = w_i * synthesis of d with m >= 1 halved    ("inverse" tables)
                        const double dm = m ? 2.0 : 1.0;
                        pf[(pf_off[m * 2 + p] + lp) * Rp + r] = static_cast<float>(v * dm);
                        pit[((m * 2 + p) * R + r) * static_cast<int64_t>(Lp) + lp] =
                            static_cast<float>(v * w[ia] / dm);
                    } else {
                        pf[(pf_off[m * 2 + p] + lp) * Rp + r] = static_cast<float>(v * w[ia]);
                        pit[((m * 2 + p) * R + r) * static_cast<int64_t>(Lp) + lp] = static_cast<float>(v);
                    }
                }
            }
        }
    });
    if (fwd_blo_conv()) {  // experiment knob SPH_GEMM_BLO_CONV_FWD=1: as the inverse below
        upload(pf_hi, pf);
    } else {
        std::vector<float> hi(pf.size()), lo(pf.size());
        tf32_split_host(pf.data(), pf.size(), hi.data(), lo.data());
        upload(pf_hi, hi);
        upload(pf_lo, lo);
    }
    // the inverse table raw: the inverse GEMM's converter warps split it in SMEM
    // (GroupedGemm::blo_conv: half its table TMA bytes); the SIMT anchor reads it exactly.
    // SPH_GEMM_BLO_CONV=0: host-split hi / lo tables instead
    if (inv_blo_conv()) {
        upload(pi_hi, pit);
    } else {
        std::vector<float> hi(pit.size()), lo(pit.size());
        tf32_split_host(pit.data(), pit.size(), hi.data(), lo.data());
        upload(pi_hi, hi);
        upload(pi_lo, lo);
    }
}

const GroupedGemm& ShtPlan::fwd_gemm(int64_t F) {
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = fwd_cache[F];
    if (!slot) {
        auto g = std::make_unique<GroupedGemm>();
        g->A = {nullptr, mmax * 2 * 2 * F, R, Rp};
        g->a_quad = true;  // E/O from fft_forward_fold: [g][Rp/4][2F][4]
        g->a_rows_g = 2 * F;
        g->a_groups = mmax * 2;
        g->a_kq = Rp / 4;
        g->Bhi = {pf_hi.p, pf_rows, R, Rp};
        g->Blo = {pf_lo.p, pf_rows, R, Rp};
        g->blo_conv = pf_lo.p == nullptr;
        g->store = STORE_ROW;
        g->bn = 192;  // TMEM-resident A operand variant
        g->name = "gemm_legendre_fwd";
        for (int64_t m = 0; m < mmax; ++m)
            for (int p = 0; p < 2; ++p) {
                const int64_t Lmp = L(m, p);
                if (Lmp == 0) continue;
                GemmGroup gr;
                gr.a_row0 = static_cast<int32_t>((m * 2 + p) * 2 * F);
                gr.b_row0 = static_cast<int32_t>(pf_off[m * 2 + p]);
                gr.M = static_cast<int32_t>(2 * F);
                gr.N = static_cast<int32_t>(Lmp);
                gr.K = R;
                gr.ldd = Lp;
                gr.zero_to = static_cast<int32_t>(std::min<int64_t>(Lp, round_up(Lmp, 8)));
                gr.d_off = (m * 2 + p) * 2 * F * Lp;
                g->groups.push_back(gr);
            }
        require(mmax * 2 * 2 * F < (1LL << 31), "sht: too many fields for one call");
        g->finalize();
        slot = std::move(g);
    }
    return *slot;
}

const GroupedGemm& ShtPlan::inv_gemm(int64_t F) {
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = inv_cache[F];
    if (!slot) {
        auto g = std::make_unique<GroupedGemm>();
        g->A = {nullptr, mmax * 2 * 2 * F, Lmax_p, Lp};
        g->Bhi = {pi_hi.p, mmax * 2 * R, Lmax_p, Lp};
        g->Blo = {pi_lo.p, mmax * 2 * R, Lmax_p, Lp};
        g->blo_conv = pi_lo.p == nullptr;
        g->store = STORE_TRANS;  // EOi[r][2F/32][m, parity][32] (fft.cu UnfoldIO)
        g->d_mode = 1;
        g->d_t = (2 * F + EOI_TILE - 1) / EOI_TILE;
        g->d_g2 = 2 * msynth;
        g->bn = 192;  // TMEM-resident A operand variant
        g->name = "gemm_legendre_inv";
        for (int64_t m = 0; m < msynth; ++m)
            for (int p = 0; p < 2; ++p) {
                const int64_t Lmp = L(m, p);
                if (Lmp == 0) continue;
                GemmGroup gr;
                gr.a_row0 = static_cast<int32_t>((m * 2 + p) * 2 * F);
                gr.b_row0 = static_cast<int32_t>((m * 2 + p) * R);
                gr.M = static_cast<int32_t>(2 * F);
                gr.N = R;
                gr.K = static_cast<int32_t>(Lmp);
                gr.ldd = static_cast<int32_t>(2 * F);
                gr.zero_to = 0;
                gr.d_off = (m * 2 + p) * 2 * F * static_cast<int64_t>(R);
                g->groups.push_back(gr);
            }
        require(mmax * 2 * 2 * F < (1LL << 31), "sht: too many fields for one call");
        g->finalize();
        slot = std::move(g);
    }
    return *slot;
}

const GroupedGemm& ShtPlan::stage_gemm(int64_t F, int64_t m0, int64_t mcount) {
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = stage_cache[std::make_tuple(F, m0, mcount)];
    if (!slot) {
        auto g = std::make_unique<GroupedGemm>();
        g->A = {nullptr, mcount * 2 * 2 * F, R, Rp};
        g->a_quad = true;  // E/O from fold_bins_kernel: [g][Rp/4][2F][4]
        g->a_rows_g = 2 * F;
        g->a_groups = mcount * 2;
        g->a_kq = Rp / 4;
        g->Bhi = {pf_hi.p, pf_rows, R, Rp};
        g->Blo = {pf_lo.p, pf_rows, R, Rp};
        g->blo_conv = pf_lo.p == nullptr;
        g->store = STORE_ROW;
        g->bn = 192;  // TMEM-resident A operand variant
        for (int64_t ml = 0; ml < mcount; ++ml)
            for (int p = 0; p < 2; ++p) {
                const int64_t m = m0 + ml;
                const int64_t Lmp = L(m, p);
                if (Lmp == 0) continue;
                GemmGroup gr;
                gr.a_row0 = static_cast<int32_t>((ml * 2 + p) * 2 * F);
                gr.b_row0 = static_cast<int32_t>(pf_off[m * 2 + p]);
                gr.M = static_cast<int32_t>(2 * F);
                gr.N = static_cast<int32_t>(Lmp);
                gr.K = R;
                gr.ldd = Lp;
                gr.zero_to = static_cast<int32_t>(std::min<int64_t>(Lp, round_up(Lmp, 8)));
                gr.d_off = (ml * 2 + p) * 2 * F * Lp;
                g->groups.push_back(gr);
            }
        g->finalize();
        slot = std::move(g);
    }
    return *slot;
}

void* ShtPlan::workspace(void* ws, int64_t bytes) {
    if (ws) return ws;
    std::lock_guard<std::mutex> lk(mu);
    if (own_ws.n < static_cast<size_t>(bytes)) own_ws.alloc(bytes, true);
    return own_ws.p;
}

void ShtPlan::forward(const float* x, int64_t F, float* out, int layout, void* ws, cudaStream_t st,
                      RingRows rr) {
    require(kind == SPH_GAUSSIAN || (flags & (SPH_FLAG_ALLOW_EQUIANGULAR_FORWARD | SPH_FLAG_ADJOINT)),
            "sht_forward: requires a gaussian grid");
    require(nlat >= lmax && nlon >= 2 * mmax, "sht_forward: resolution insufficient for lmax/mmax");
    require(layout == SPH_LAYOUT_DENSE_LM || layout == SPH_LAYOUT_INTERNAL, "sht_forward: bad layout");
    require(F >= 0, "sht_forward: negative field count");
    if (F == 0) return;
    DeviceGuard dguard(device);
    require_on_device(x, device, "sht_forward");
    require_on_device(out, device, "sht_forward");
    uint8_t* w8 = static_cast<uint8_t*>(workspace(ws, workspace_bytes(F)));
    float* eo = reinterpret_cast<float*>(w8);
    float* ctmp = reinterpret_cast<float*>(w8 + round_up(4 * eo_elems(F), 256));
    fft_forward_fold(fft, fold, x, F, static_cast<int>(nlat), static_cast<int>(mmax), eo, Rp, st, rr);
    float* target = layout == SPH_LAYOUT_INTERNAL ? out : ctmp;
    gemm_run(fwd_gemm(F), eo, target, prec, st);
    if (layout == SPH_LAYOUT_DENSE_LM) cint_to_dense(*this, target, F, 0, mmax, mmax, out, st);
}

void ShtPlan::inverse(const float* coeffs, int64_t F, int layout, float* y, void* ws,
                      cudaStream_t st, RingRows rr) {
    require(layout == SPH_LAYOUT_DENSE_LM || layout == SPH_LAYOUT_INTERNAL, "sht_inverse: bad layout");
    require(F >= 0, "sht_inverse: negative field count");
    if (F == 0) return;
    DeviceGuard dguard(device);
    require_on_device(coeffs, device, "sht_inverse");
    require_on_device(y, device, "sht_inverse");
    uint8_t* w8 = static_cast<uint8_t*>(workspace(ws, workspace_bytes(F)));
    float* eoi = reinterpret_cast<float*>(w8);
    float* ctmp = reinterpret_cast<float*>(w8 + round_up(4 * eo_elems(F), 256));
    const float* src = coeffs;
    if (layout == SPH_LAYOUT_DENSE_LM) {
        dense_to_cint(*this, coeffs, F, ctmp, st);
        src = ctmp;
    }
    gemm_run(inv_gemm(F), src, eoi, prec, st);
    fft_inverse_unfold(fft, fold, eoi, F, static_cast<int>(nlat), static_cast<int>(mmax),
                       static_cast<int>(msynth), static_cast<int>(lmax), Rp, y, st, rr);
}

void ShtPlan::fft_stage(const float* rings, int64_t F, int64_t h, float* bins, cudaStream_t st) {
    require(nlon >= 2 * mmax, "dist_sht_forward: resolution insufficient for mmax");
    DeviceGuard dguard(device);
    const double pi = 3.14159265358979323846;
    fft_forward_plain(fft, rings, F * h, static_cast<int>(mmax),
                      static_cast<float>(2.0 * pi / static_cast<double>(nlon)),
                      reinterpret_cast<float2*>(bins), st);
}

void ShtPlan::legendre_stage(const float* bins, int64_t F, int64_t m0, int64_t mcount,
                             float* coeffs, void* ws, cudaStream_t st) {
    require(m0 >= 0 && mcount >= 0 && m0 + mcount <= mmax, "legendre stage: order range");
    require(nlat >= lmax, "dist_sht_forward: resolution insufficient for lmax");
    if (F == 0 || mcount == 0) return;
    DeviceGuard dguard(device);
    uint8_t* w8 = static_cast<uint8_t*>(workspace(ws, stage_ws_bytes(F, mcount)));
    float* eo = reinterpret_cast<float*>(w8);
    float* cl = reinterpret_cast<float*>(w8 + round_up(4 * mcount * 2 * 2 * F * Rp, 256));
    const int64_t n = mcount * 2 * 2 * F * Rp;
    const double pi = 3.14159265358979323846;
    fold_bins_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const float2*>(bins), fold.d_rows.p, R, Rp, F, nlat, mcount,
        static_cast<float>(static_cast<double>(nlon) / (2.0 * pi)), eo);
    SPH_LAUNCH_CHECK();
    count_launch();
    gemm_run(stage_gemm(F, m0, mcount), eo, cl, prec, st);
    cint_to_dense(*this, cl, F, m0, mcount, mcount, coeffs, st);
}

// ------------------------------------------------------------- host round trip
// Three streams: uploads (H2D), compute (forward + inverse SHT), downloads (D2H), and
// NB chunk buffers.  Chunk i uses buffer i % NB; its upload waits until the compute of
// chunk i - NB has consumed x[s], its compute waits for its upload and for the download
// of chunk i - NB (y[s] free).  H2D and D2H of different chunks then run concurrently on
// the two copy engines (measured 89 GB/s combined vs 55 GB/s one way on a Gen5 x16 link),
// and streams / buffers persist across calls (the former per-call 2-stream version
// allocated ~2 GB and serialised each chunk's upload behind the previous download).
struct ShtPlan::HostPipe {
    static constexpr int NB = 3;
    int64_t chunk = 0;
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t up[NB], used[NB], down[NB];
    DevBuf<float> x[NB], y[NB], c;
    DevBuf<uint8_t> ws;
    HostPipe(ShtPlan& p, int64_t ch) : chunk(ch) {
        SPH_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
        SPH_CUDA(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking));
        SPH_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
        const int64_t np = p.nlat * p.nlon;
        for (int i = 0; i < NB; ++i) {
            SPH_CUDA(cudaEventCreateWithFlags(&up[i], cudaEventDisableTiming));
            SPH_CUDA(cudaEventCreateWithFlags(&used[i], cudaEventDisableTiming));
            SPH_CUDA(cudaEventCreateWithFlags(&down[i], cudaEventDisableTiming));
            x[i].alloc(ch * np, false);
            y[i].alloc(ch * np, false);
        }
        c.alloc(p.cint_elems(ch), true);
        ws.alloc(p.workspace_bytes(ch), true);
    }
    ~HostPipe() {
        for (int i = 0; i < NB; ++i) {
            cudaEventDestroy(up[i]);
            cudaEventDestroy(used[i]);
            cudaEventDestroy(down[i]);
        }
        cudaStreamDestroy(h2d);
        cudaStreamDestroy(comp);
        cudaStreamDestroy(d2h);
    }
};

ShtPlan::ShtPlan() = default;
ShtPlan::~ShtPlan() = default;

void ShtPlan::roundtrip_host(const float* xh, int64_t F, float* yh, int64_t chunk) {
    if (F <= 0) return;
    DeviceGuard dguard(device);
    if (chunk <= 0) chunk = 32;
    chunk = std::min(chunk, F);
    std::lock_guard<std::mutex> lk(pipe_mu);  // one round trip per plan at a time
    if (!pipe || pipe->chunk != chunk) {
        if (pipe) SPH_CUDA(cudaDeviceSynchronize());
        pipe = std::make_unique<HostPipe>(*this, chunk);
    }
    HostPipe& q = *pipe;
    const int64_t np = nlat * nlon;
    int it = 0;
    for (int64_t f0 = 0; f0 < F; f0 += chunk, ++it) {
        const int s = it % HostPipe::NB;
        const int64_t n = std::min(chunk, F - f0);
        if (it >= HostPipe::NB) SPH_CUDA(cudaStreamWaitEvent(q.h2d, q.used[s], 0));
        SPH_CUDA(cudaMemcpyAsync(q.x[s].p, xh + f0 * np, sizeof(float) * n * np, cudaMemcpyHostToDevice,
                                 q.h2d));
        SPH_CUDA(cudaEventRecord(q.up[s], q.h2d));
        SPH_CUDA(cudaStreamWaitEvent(q.comp, q.up[s], 0));
        if (it >= HostPipe::NB) SPH_CUDA(cudaStreamWaitEvent(q.comp, q.down[s], 0));
        forward(q.x[s].p, n, q.c.p, SPH_LAYOUT_INTERNAL, q.ws.p, q.comp);
        SPH_CUDA(cudaEventRecord(q.used[s], q.comp));
        inverse(q.c.p, n, SPH_LAYOUT_INTERNAL, q.y[s].p, q.ws.p, q.comp);
        SPH_CUDA(cudaEventRecord(q.up[s], q.comp));  // reuse: "computed"
        SPH_CUDA(cudaStreamWaitEvent(q.d2h, q.up[s], 0));
        SPH_CUDA(cudaMemcpyAsync(yh + f0 * np, q.y[s].p, sizeof(float) * n * np, cudaMemcpyDeviceToHost,
                                 q.d2h));
        SPH_CUDA(cudaEventRecord(q.down[s], q.d2h));
    }
    SPH_CUDA(cudaStreamSynchronize(q.d2h));
}

}  // namespace sph
