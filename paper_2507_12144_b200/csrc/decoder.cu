// Fused decoder: bilinear upsampling (resample.hpp:20-114) folded into the decoder's
// DISCO convolution (convolution.hpp:181-220) in the longitude-Fourier domain.
//
// DISCO's Fourier path starts from the channel-minor half spectrum U[b][h][m][c] of its
// input rings.  When the output ring length is an integer multiple r of the latent one,
// the upsampled ring is the latent ring zero-stuffed by r and convolved with the periodic
// hat (1 - |d|/r, |d| < r), so its spectrum is
//     U_row(m) = H(m) * [(1 - wt) X_i0(m mod n_lat) + wt X_i1(m mod n_lat)],
//     H(m) = (1/r) (sin(pi m r / n_out) / sin(pi m / n_out))^2,   H(0) = r
// with X_i the latent ring spectrum (Hermitian extension above n_lat/2) and the
// pole-extension rows, constant rings of the first / last ring mean, contributing only
// their DC bin X_0(0) / X_{H-1}(0).  The decoder therefore runs the R2C on the latent
// rings (r x fewer samples), builds U directly (one gather pass, HBM-bound: 2 complex reads
// + 1 complex write per output bin per channel) and hands it to DISCO's band / mix / C2R
// stages; the upsampled field is never materialized.  Otherwise (non-integer ratio, or the
// direct-gather SIMT precision) the upsampled field is materialized and convolved.
#include <algorithm>
#include <cmath>

#include "decoder.cuh"

namespace sph {
namespace {
constexpr double kPi = 3.14159265358979323846;

// thread per (bin m, channel group): V = float4 carries a channel pair (even channel
// counts, both spectra in the pair-interleaved layout), float2 one channel
__device__ __forceinline__ float4 vzero(float4) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float2 vzero(float2) { return make_float2(0.f, 0.f); }
// float4 = channel pair in DISCO's pair-interleaved layout (re c, re c+1, im c, im c+1)
__device__ __forceinline__ void vconj(float4& v) { v.z = -v.z; v.w = -v.w; }
__device__ __forceinline__ void vconj(float2& v) { v.y = -v.y; }
__device__ __forceinline__ float4 vaxpby(float a, float4 p, float b, float4 q) {
    return make_float4(fmaf(b, q.x, a * p.x), fmaf(b, q.y, a * p.y), fmaf(b, q.z, a * p.z), fmaf(b, q.w, a * p.w));
}
__device__ __forceinline__ float2 vaxpby(float a, float2 p, float b, float2 q) {
    return make_float2(fmaf(b, q.x, a * p.x), fmaf(b, q.y, a * p.y));
}

template <class V>
__global__ void fourier_upsample_kernel(const V* __restrict__ UL, int HL, int nbl, int nl, int HO, int nbo, int CV,
                                        const int32_t* __restrict__ i0s, const int32_t* __restrict__ i1s,
                                        const float* __restrict__ wts, int row0, int north, int south,
                                        const float* __restrict__ hm, V* __restrict__ U) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nbo * CV) return;
    const int m = t / CV;
    const int c = t - m * CV;
    const int oi = blockIdx.y, b = blockIdx.z;
    const int k = m % nl;
    const bool cj = k > nl / 2;
    const int kk = cj ? nl - k : k;
    // spectrum bin k of extended latent row er
    auto X = [&](int er) -> V {
        int ring, bin = kk;
        if (er == north || er == south) {
            if (k != 0) return vzero(V{});
            ring = er == north ? 0 : HL - 1;
            bin = 0;
        } else {
            ring = er - row0;
        }
        V v = __ldg(UL + ((static_cast<int64_t>(b) * HL + ring) * nbl + bin) * CV + c);
        if (cj && bin) vconj(v);
        return v;
    };
    const float wt = wts[oi];
    const float h = hm[m];
    const V p = X(i0s[oi]);
    const V q = wt != 0.f ? X(i1s[oi]) : vzero(V{});
    U[((static_cast<int64_t>(b) * HO + oi) * nbo + m) * CV + c] = vaxpby(h * (1.f - wt), p, h * wt, q);
}
}  // namespace

void DecoderPlan::create(DiscoPlan* d, const double* lat_colat, int64_t lat_nlat, int64_t lat_nlon) {
    require(d != nullptr, "decode: null DISCO plan");
    require(d->hin == d->hout && d->win == d->wout && d->stride == 1,
            "decode: the decoder convolution maps the output grid onto itself");
    disco = d;
    DeviceGuard dguard(d->device);
    resample_create(rs, lat_colat, lat_nlat, lat_nlon, d->in_colat.data(), d->hin, d->win);
    ratio = static_cast<int>(d->win / lat_nlon);
    fourier = d->prec != SPH_PREC_FP32_SIMT && d->win % lat_nlon == 0 && lat_nlon <= (1 << 30);
    if (!fourier) return;
    fft_lat.build(static_cast<int>(lat_nlon));
    nbl = lat_nlon / 2 + 1;
    // exact positions: output column oj sits at latent position oj / r (resample.hpp:92-105
    // snaps to these within 1e-12), so the plan's column brackets are the hat interpolant
    for (int64_t oj = 0; oj < d->win; ++oj)
        require(rs.j0[oj] == oj / ratio && std::fabs(rs.wp[oj] - static_cast<double>(oj % ratio) / ratio) < 1e-9,
                "decode: unexpected longitude brackets");
    std::vector<float> h(d->nbi);
    for (int64_t m = 0; m < d->nbi; ++m) {
        if (m == 0) {
            h[m] = static_cast<float>(ratio);
            continue;
        }
        const double s1 = std::sin(kPi * static_cast<double>(m) * ratio / static_cast<double>(d->win));
        const double s0 = std::sin(kPi * static_cast<double>(m) / static_cast<double>(d->win));
        h[m] = static_cast<float>(s1 * s1 / (s0 * s0) / ratio);
    }
    d_h.alloc(h.size(), false);
    SPH_CUDA(cudaMemcpy(d_h.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
}

namespace {
struct DecWs {
    int64_t disco, extra_off, total;
};
DecWs dec_ws(const DecoderPlan& p, int64_t B, int64_t cin, int64_t cout) {
    DecWs w;
    w.disco = static_cast<int64_t>(round_up(static_cast<size_t>(p.disco->workspace_bytes(B, cin, cout)), 256));
    w.extra_off = w.disco;
    int64_t extra;
    if (p.fourier)
        extra = B * p.rs.in_nlat * p.nbl * cin * static_cast<int64_t>(sizeof(float2));
    else
        extra = static_cast<int64_t>(round_up(static_cast<size_t>(B * cin * p.disco->hin * p.disco->win * 4), 256)) +
                resample_workspace_bytes(p.rs, B * cin);
    w.total = w.disco + static_cast<int64_t>(round_up(static_cast<size_t>(extra), 256));
    return w;
}
}  // namespace

int64_t DecoderPlan::workspace_bytes(int64_t B, int64_t cin, int64_t cout) const {
    return dec_ws(*this, B, cin, cout).total;
}

void DecoderPlan::apply(const float* latent, const float* mix, int64_t B, int64_t cin, int64_t cout, float* y,
                        void* ws, cudaStream_t st) {
    require(B >= 0 && cin >= 1 && cout >= 1, "decode: mix tensor shape mismatch");
    if (B == 0) return;
    DeviceGuard dguard(disco->device);
    const DecWs w = dec_ws(*this, B, cin, cout);
    uint8_t* base = static_cast<uint8_t*>(ws);
    if (!base) {
        std::lock_guard<std::mutex> lk(mu);
        if (own_ws.n < static_cast<size_t>(w.total)) own_ws.alloc(w.total, true);
        base = own_ws.p;
    }
    uint8_t* extra = base + w.extra_off;
    if (!fourier) {
        float* up = reinterpret_cast<float*>(extra);
        void* rws = extra + round_up(static_cast<size_t>(B * cin * disco->hin * disco->win * 4), 256);
        resample_apply(rs, latent, B * cin, up, rws, st);
        disco->apply(up, mix, B, cin, cout, y, base, st);
        return;
    }
    require(B <= 65535 && disco->hin <= 65535, "decode: grid too large");
    float2* UL = reinterpret_cast<float2*>(extra);
    const int64_t HL = rs.in_nlat, HO = disco->hin;
    const int row0 = rs.add_north ? 1 : 0;
    const int north = rs.add_north ? 0 : -1, south = rs.add_south ? static_cast<int>(rs.ext_nlat - 1) : -1;
    const std::function<void(float2*)> make_u = [&](float2* U) {
        const bool pairs = disco->pair_layout(cin);
        fft_forward_cminor(fft_lat, latent, B, cin, HL, static_cast<int>(nbl), UL, st, pairs ? 2 : 0);
        const int CV = static_cast<int>(pairs ? cin / 2 : cin);
        const int64_t n = disco->nbi * CV;
        dim3 grid(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(HO), static_cast<unsigned>(B));
        {
            ProfScope prof("decoder_upsample", st, 8.0 * B * (HL * nbl * cin + 2 * HO * disco->nbi * cin));
            auto go = [&](auto* ul, auto* u) {
                fourier_upsample_kernel<<<grid, 256, 0, st>>>(
                    ul, static_cast<int>(HL), static_cast<int>(nbl), static_cast<int>(rs.in_nlon),
                    static_cast<int>(HO), static_cast<int>(disco->nbi), CV, rs.d_i0.p, rs.d_i1.p, rs.d_wt.p, row0,
                    north, south, d_h.p, u);
            };
            if (pairs)
                go(reinterpret_cast<const float4*>(UL), reinterpret_cast<float4*>(U));
            else
                go(static_cast<const float2*>(UL), U);
            SPH_LAUNCH_CHECK();
        }
        count_launch();
    };
    disco->apply_rows(nullptr, 0, HO, 0, disco->hout, mix, B, cin, cout, y, base, st, &make_u);
}

}  // namespace sph
