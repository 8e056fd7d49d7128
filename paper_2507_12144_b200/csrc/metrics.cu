// SHT consumers on sm_100a: angular power spectrum (metrics.hpp:300-314)
// and the spectral CRPS loss (loss.hpp:37-81), as reductions over the dense coefficient
// layout [F][lmax][mmax] complex produced by sph_sht_forward.
#include "metrics.cuh"

namespace sph {
namespace {

// psd[f][l] = |c(l,0)|^2 + 2 sum_{1 <= m <= min(l, mmax-1)} |c(l,m)|^2   (fp64 accumulation)
__global__ void psd_kernel(const float2* __restrict__ c, int64_t F, int64_t lmax, int64_t mmax,
                           float* __restrict__ psd) {
    const int64_t f = blockIdx.y;
    const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
    if (l >= lmax) return;
    const float2* row = c + (f * lmax + l) * mmax;
    const int64_t mt = min(l, mmax - 1);
    double s = 0.0;
    for (int64_t m = threadIdx.x; m <= mt; m += 32) {
        const float2 v = row[m];
        const double n = static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y;
        s += m == 0 ? n : 2.0 * n;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) psd[f * lmax + l] = static_cast<float>(s);
}

// one thread per (c, l, m, re/im): ensemble CRPS of the E member coefficients against the
// observation (metrics.hpp:160-209); cdf and spread_skill are the same integral (biased),
// fair divides the spread term by 2N(N-1).  The pairwise sum is formed exactly in O(E^2).
__global__ void spectral_crps_kernel(const float2* __restrict__ ens, const float2* __restrict__ obs, int E,
                                     int64_t C, int64_t lmax, int64_t mmax, int64_t lmax_sum, int fair,
                                     double* __restrict__ out) {
    const int64_t per_c = lmax_sum * mmax * 2;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t c = blockIdx.y;
    double v = 0.0;
    if (i < per_c) {
        const int ri = static_cast<int>(i & 1);
        const int64_t m = (i >> 1) % mmax;
        const int64_t l = 1 + (i >> 1) / mmax;
        if (m <= min(l, mmax - 1)) {
            constexpr int EMAX = 64;
            float u[EMAX];
            const int64_t stride = C * lmax * mmax;
            const int64_t off = (c * lmax + l) * mmax + m;
            for (int e = 0; e < E; ++e) {
                const float2 z = ens[e * stride + off];
                u[e] = ri ? z.y : z.x;
            }
            const float2 zo = obs[off];
            const double o = ri ? zo.y : zo.x;
            double skill = 0.0, pair = 0.0;
            for (int e = 0; e < E; ++e) {
                skill += fabs(static_cast<double>(u[e]) - o);
                for (int k = e + 1; k < E; ++k) pair += fabs(static_cast<double>(u[e]) - static_cast<double>(u[k]));
            }
            const double n = E;
            skill /= n;
            const double denom = fair ? 2.0 * n * (n - 1.0) : 2.0 * n * n;
            const double crps = skill - 2.0 * pair / denom;
            v = (m == 0 ? 1.0 : 2.0) * crps;
        }
    }
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v != 0.0) atomicAdd(out + c, v);
}

// dist_crps local kernel (distsim.hpp:591-618): thread per (channel, spatial sample k):
// ensemble CRPS of f[e][c][k] against o[c][k], times w[k] (quadrature weight of the
// sample's latitude), summed per channel in fp64 and divided by 4 pi.
__global__ void weighted_crps_kernel(const float* __restrict__ f, const float* __restrict__ o,
                                     const float* __restrict__ w, int E, int64_t C, int64_t ns, int fair,
                                     double* __restrict__ out) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t c = blockIdx.y;
    double v = 0.0;
    if (k < ns) {
        constexpr int EMAX = 64;
        float u[EMAX];
        for (int e = 0; e < E; ++e) u[e] = f[(e * C + c) * ns + k];
        const double ob = o[c * ns + k];
        double skill = 0.0, pair = 0.0;
        for (int e = 0; e < E; ++e) {
            skill += fabs(static_cast<double>(u[e]) - ob);
            for (int q = e + 1; q < E; ++q) pair += fabs(static_cast<double>(u[e]) - static_cast<double>(u[q]));
        }
        const double n = E;
        const double denom = fair ? 2.0 * n * (n - 1.0) : 2.0 * n * n;
        v = static_cast<double>(w[k]) * (skill / n - 2.0 * pair / denom) / (4.0 * 3.14159265358979323846);
    }
    for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
    if ((threadIdx.x & 31) == 0 && v != 0.0) atomicAdd(out + c, v);
}

}  // namespace

void weighted_crps(const float* f, const float* o, const float* w, int64_t E, int64_t C, int64_t ns, int variant,
                   double* out, cudaStream_t st) {
    require(E >= 1 && E <= 64, "dist_crps: 1..64 ensemble members supported");
    require(variant >= 0 && variant <= 2, "dist_crps: unknown CRPS variant");
    require(variant != 2 || E >= 2, "crps_pointwise: fair variant needs E >= 2");
    require(C <= 65535, "dist_crps: too many channels");
    SPH_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * C, st));
    if (C == 0 || ns == 0) return;
    dim3 grid(static_cast<unsigned>((ns + 255) / 256), static_cast<unsigned>(C));
    weighted_crps_kernel<<<grid, 256, 0, st>>>(f, o, w, static_cast<int>(E), C, ns, variant == 2 ? 1 : 0, out);
    SPH_LAUNCH_CHECK();
    count_launch();
}

void psd_from_coeffs(const float* coeffs, int64_t F, int64_t lmax, int64_t mmax, float* psd, cudaStream_t st) {
    require(F >= 0 && lmax >= 1 && mmax >= 1, "angular_psd: bad shapes");
    if (F == 0) return;
    require(F <= 65535, "angular_psd: at most 65535 fields per call");
    dim3 grid(static_cast<unsigned>((lmax + 7) / 8), static_cast<unsigned>(F));
    psd_kernel<<<grid, dim3(32, 8), 0, st>>>(reinterpret_cast<const float2*>(coeffs), F, lmax, mmax, psd);
    SPH_LAUNCH_CHECK();
    count_launch();
}

void spectral_crps_from_coeffs(const float* ens, const float* obs, int64_t E, int64_t C, int64_t lmax,
                               int64_t mmax, int64_t lmax_sum, int variant, double* out, cudaStream_t st) {
    require(E >= 1 && E <= 64, "spectral_crps_loss: 1..64 ensemble members supported");
    require(variant >= 0 && variant <= 2, "spectral_crps_loss: unknown CRPS variant");
    require(variant != 2 || E >= 2, "crps_pointwise: fair variant needs E >= 2");
    require(lmax_sum >= 1 && lmax_sum + 1 <= lmax, "spectral_crps_loss: lmax_sum exceeds grid capacity");
    require(C <= 65535, "spectral_crps_loss: too many channels");
    SPH_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * C, st));
    if (C == 0) return;
    const int64_t per_c = lmax_sum * mmax * 2;
    dim3 grid(static_cast<unsigned>((per_c + 255) / 256), static_cast<unsigned>(C));
    spectral_crps_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float2*>(ens),
                                               reinterpret_cast<const float2*>(obs), static_cast<int>(E), C, lmax,
                                               mmax, lmax_sum, variant == 2 ? 1 : 0, out);
    SPH_LAUNCH_CHECK();
    count_launch();
}

}  // namespace sph
