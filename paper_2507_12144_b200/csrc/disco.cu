// DISCO convolution on sm_100a (convolution.hpp:141-220).
//
// The operator is assembled on the host in fp64 exactly as the reference does
// (every k shares one (h_in, w_rel) index list per output row; the input quadrature
// weight is folded in).  Two device paths:
//
//  * default (SPH_PREC_3XTF32 / TF32): longitude-Fourier restructure.  psi_k for a fixed
//    (h_out, h_in) pair is a circular correlation filter over the longitude index, so
//        t_hat[k,c,h](m) = sum_{h_in in band(h)} conj(psi_hat_k[h,h_in](m)) u_hat[c,h_in](m)
//    and the stride-s output sampling folds the spectrum:  S(m') = sum_q R(m' + W_out q).
//    Kernels: channel-minor R2C of the input rings -> band contraction (<= ~12 rows per
//    output row, independent of the polar row nnz) -> tcgen05 3xTF32 channel-mix GEMM
//    (mix [c_out][c_in*K] is the table operand) in the Fourier domain -> C2R of the
//    output rings.  Parity is by tolerance (summation order differs).
//  * SPH_PREC_FP32_SIMT anchor: the reference's own operation order (gather t, then
//    the channel mix) in fp32 FMA.
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <mutex>
#include <thread>

#include "disco.cuh"

namespace sph {

namespace {
constexpr double kPi = 3.14159265358979323846;
}

int Basis::n_real() const {
    int n = 0;
    for (auto& p : pairs) n += (p.first == 0 && p.second == 0) ? 1 : 2;
    return n;
}

// convolution.hpp:38-68 (Hann-windowed Morlet modes, real then imaginary parts)
double Basis::eval_real(int k, double theta, double phi) const {
    size_t b = 0;
    for (; b < pairs.size(); ++b) {
        const int parts = (pairs[b].first == 0 && pairs[b].second == 0) ? 1 : 2;
        if (k < parts) break;
        k -= parts;
    }
    const double tp = theta / cutoff;
    if (tp > 1.0) return 0.0;
    const double c = std::cos(0.5 * kPi * tp);
    const double h = c * c;
    const double arg = kPi * tp * (pairs[b].first * std::sin(phi) + pairs[b].second * std::cos(phi));
    return k == 0 ? h * std::cos(arg) : h * std::sin(arg);
}

Basis make_basis(int kind, double cutoff) {
    require(cutoff > 0.0, kind == SPH_BASIS_ISOTROPIC ? "isotropic_basis: cutoff must be > 0"
                                                      : "morlet_basis: cutoff must be > 0");
    Basis b;
    b.cutoff = cutoff;
    if (kind == SPH_BASIS_MORLET)
        b.pairs = {{0, 0}, {0, 1}, {0, 2}, {2, 1}, {2, 2}};  // convolution.hpp:73-76
    else if (kind == SPH_BASIS_ISOTROPIC)
        b.pairs = {{0, 0}};
    else
        fail(SPH_ERR_INVALID_ARGUMENT, "disco: unknown basis");
    return b;
}

namespace {

// convolution.hpp:93-101: great-circle distance and azimuth from the southward meridian
inline void chart(double theta_out, double theta_in, double dphi, double& dist, double& az) {
    const double st_o = std::sin(theta_out), ct_o = std::cos(theta_out);
    const double st_i = std::sin(theta_in), ct_i = std::cos(theta_in);
    const double cd = std::cos(dphi);
    const double x = ct_o * st_i * cd - st_o * ct_i;
    const double y = st_i * std::sin(dphi);
    const double z = st_o * st_i * cd + ct_o * ct_i;
    dist = std::atan2(std::hypot(x, y), z);
    az = std::atan2(y, x);
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
    d.alloc(std::max<size_t>(h.size(), 1), false);
    if (!h.empty()) SPH_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

// ---------------------------------------------------------------- kernels
__global__ void split_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t cols,
                                  int64_t ld, float* __restrict__ hi, float* __restrict__ lo) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows * ld) return;
    const int64_t r = i / ld, c = i % ld;
    const float x = c < cols ? src[r * cols + c] : 0.f;
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    const float h = __uint_as_float(u);
    hi[i] = h;
    lo[i] = x - h;
}

// threads = (m' in tile) x 64 channel lanes; the CTA loops over the batch.  The psi_hat
// slice of the block (band rows x folds x 4 orders x K) and each slot's U row offset +
// Hermitian-fold flag are staged in shared memory once per slot chunk, so the inner loop
// is 1 LDG + 5 broadcast LDS.128 + 36 FFMA per slot (the former per-slot integer
// decoding made it instruction-issue bound: FFMA 13 % of instructions, issue 63 %).
// Batch register blocking (2 or 4 batches per thread) was measured slower (spills).
// Output S[((b*Hout + h)*nbo + m')*2 + reim][c*K + k].
constexpr int BAND_MAX_SLOTS = 64;  // band rows x folds staged per CTA
__global__ void __launch_bounds__(256) disco_band_kernel(
    const float2* __restrict__ U, const float2* __restrict__ psi_hat, const int32_t* __restrict__ band0,
    const int32_t* __restrict__ bandc, const int64_t* __restrict__ psi_off, int64_t Hin, int64_t nbi,
    int64_t Hout, int64_t nbo, int win, int wout, int s, int K, int64_t C, int64_t ldS,
    float* __restrict__ S, int64_t h_in0, int64_t ho0, int64_t B) {
    // U holds input rows [h_in0, h_in0 + Hin); this launch computes output rows
    // [ho0, ho0 + Hout) (local index h)
    __shared__ float4 ps[BAND_MAX_SLOTS][4][5];  // [band slot][m' in tile][k pairs] (K <= 9 -> 5 float4)
    __shared__ int32_t uo[BAND_MAX_SLOTS][4];    // (bi * nbi + idx), ~x when folded (conj)
    __shared__ __align__(16) float so[4][2][64 * 9];  // output tile [m'][re, im][c * K + k]
    const int mi = threadIdx.x / 64, cl = threadIdx.x % 64;
    const int64_t mp0 = static_cast<int64_t>(blockIdx.x) * 4;
    const int64_t mp = mp0 + mi;
    const int64_t h = blockIdx.y;
    const int64_t hg = ho0 + h;
    const int h0 = band0[hg] - static_cast<int>(h_in0), nb = bandc[hg];
    const int64_t po = psi_off[hg];
    const int half = win / 2;
    const int nslot = nb * s;
    for (int slot0 = 0; slot0 < nslot; slot0 += BAND_MAX_SLOTS) {
        const int ns = min(BAND_MAX_SLOTS, nslot - slot0);
        __syncthreads();
        for (int i = threadIdx.x; i < ns * 4 * 10; i += blockDim.x) {
            const int kk = i % 10, t = (i / 10) % 4, sl = i / 40;
            const int slot = slot0 + sl;
            const int bi = slot / s, q = slot - bi * s;
            const int64_t m = mp0 + t;
            float2 v = make_float2(0.f, 0.f);
            const int kq = static_cast<int>(m) + wout * q;
            const int idx = kq > half ? win - kq : kq;
            if (m < nbo && kk < K) v = __ldg(psi_hat + ((po + bi) * nbi + idx) * K + kk);
            reinterpret_cast<float2*>(&ps[sl][t][0])[kk] = v;
            if (kk == 0) {
                const int o = bi * static_cast<int>(nbi) + (m < nbo ? idx : 0);
                uo[sl][t] = kq > half ? ~o : o;
            }
        }
        __syncthreads();
        const bool mact = mp < nbo;
        for (int64_t b = 0; b < B; ++b) {
            for (int64_t c0 = 0; c0 < C; c0 += 64) {
                const int64_t c = c0 + cl;
                const int cn = static_cast<int>(C - c0 < 64 ? C - c0 : 64);
                float2 acc[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[k] = make_float2(0.f, 0.f);
                if (mact && c < C) {
                const float2* Ub = U + (b * Hin + h0) * nbi * C + c;
                // slots in batches of 4 with the next batch's U loads in flight while the
                // current batch is consumed (the loop was load-latency bound: long
                // scoreboard 57 % of stalls)
                constexpr int CH = 4;
                float2 ucur[CH], unxt[CH];
                int ocur[CH], onxt[CH];
                auto load = [&](int sl0, float2 (&u)[CH], int (&o)[CH]) {
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        const int sl = sl0 + j;
                        o[j] = sl < ns ? uo[sl][mi] : 0;
                        const int oo = o[j] < 0 ? ~o[j] : o[j];
                        u[j] = sl < ns ? __ldg(Ub + static_cast<int64_t>(oo) * C) : make_float2(0.f, 0.f);
                    }
                };
                load(0, ucur, ocur);
                for (int sl0 = 0; sl0 < ns; sl0 += CH) {
                    if (sl0 + CH < ns) load(sl0 + CH, unxt, onxt);
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        if (sl0 + j >= ns) break;
                        const float4* pp = &ps[sl0 + j][mi][0];
                        float2 p[10];
#pragma unroll
                        for (int k2 = 0; k2 < 5; ++k2) {
                            const float4 t4 = pp[k2];
                            p[2 * k2] = make_float2(t4.x, t4.y);
                            p[2 * k2 + 1] = make_float2(t4.z, t4.w);
                        }
                        // R = conj(psi) u for kq <= W/2, psi conj(u) = conj(conj(psi) u)
                        // above (Hermitian fold): re += px ux + py uy, im += px vx - py vy
                        // with (vx, vy) = sy * (uy, ux)
                        const bool cj = ocur[j] < 0;
                        const float ux = ucur[j].x, uy = ucur[j].y;
                        const float vx = cj ? -uy : uy, vy = cj ? -ux : ux;
#pragma unroll
                        for (int k = 0; k < 9; ++k) {
                            acc[k].x = fmaf(p[k].x, ux, fmaf(p[k].y, uy, acc[k].x));
                            acc[k].y = fmaf(p[k].x, vx, fmaf(-p[k].y, vy, acc[k].y));
                        }
                    }
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        ucur[j] = unxt[j];
                        ocur[j] = onxt[j];
                    }
                }
                }
                // stage the [4 m][re, im][cn * K] tile in shared memory (stride K per
                // channel: odd K = 9 -> conflict-free) and store it as contiguous rows
                __syncthreads();
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    if (k < K) {
                        so[mi][0][cl * K + k] = acc[k].x;
                        so[mi][1][cl * K + k] = acc[k].y;
                    }
                __syncthreads();
                const int rowlen = cn * K;
                const int nt = static_cast<int>(nbo - mp0 < 4 ? nbo - mp0 : 4);
                if ((rowlen & 3) == 0 && (ldS & 3) == 0 && ((c0 * K) & 3) == 0) {
                    const int q4 = rowlen >> 2;
                    for (int i = threadIdx.x; i < nt * 2 * q4; i += blockDim.x) {
                        const int r = i / q4, j = i - r * q4;
                        const int t = r >> 1, ri = r & 1;
                        const int64_t row = ((b * Hout + h) * nbo + mp0 + t) * 2 + ri;
                        float4* dst = reinterpret_cast<float4*>(S + row * ldS + c0 * K) + j;
                        float4 v = reinterpret_cast<const float4*>(&so[t][ri][0])[j];
                        if (slot0 != 0) {
                            const float4 o = *dst;
                            v.x += o.x;
                            v.y += o.y;
                            v.z += o.z;
                            v.w += o.w;
                        }
                        *dst = v;
                    }
                } else {
                    for (int i = threadIdx.x; i < nt * 2 * rowlen; i += blockDim.x) {
                        const int r = i / rowlen, j = i - r * rowlen;
                        const int t = r >> 1, ri = r & 1;
                        const int64_t row = ((b * Hout + h) * nbo + mp0 + t) * 2 + ri;
                        float* dst = S + row * ldS + c0 * K + j;
                        const float v = so[t][ri][j];
                        *dst = slot0 != 0 ? *dst + v : v;
                    }
                }
            }
        }
    }
}

// Even channel counts: each thread owns a channel pair (c, c+1) and accumulates both in
// packed fp32x2 registers with FFMA2 (fma.rn.f32x2, the psi value as a broadcast scalar
// operand): a slot costs 1 LDG.128 + 9 broadcast LDS.128 + 36 FFMA2 for 2 channels
// (the scalar kernel: 2 x (1 LDG + 5 LDS + 36 FFMA + selects)).  U arrives in the
// pair-interleaved layout (re c, re c+1, im c, im c+1), so one float4 is directly the two
// packed operands; the Hermitian-fold sign is folded into the staged psi values:
// per (slot, order, k) smem holds (px, py, s px, -s py) with
//     re += px ux + py uy,   im += s (px uy - py ux),   s = -1 for folded bins.
// threads = 4 orders x 32 lanes, 64 channels per pass.
// acc += a * b for a float2 pair with a broadcast scalar (FFMA2 R.F32 operand)
__device__ __forceinline__ void ffma2(float2& d, float a, float2 b) { d = __ffma2_rn(make_float2(a, a), b, d); }

constexpr int BAND2_SLOTS = 32;
__global__ void __launch_bounds__(128) disco_band2_kernel(
    const float4* __restrict__ U, const float2* __restrict__ psi_hat, const int32_t* __restrict__ band0,
    const int32_t* __restrict__ bandc, const int64_t* __restrict__ psi_off, int64_t Hin, int64_t nbi,
    int64_t Hout, int64_t nbo, int win, int wout, int s, int K, int64_t C, int64_t ldS,
    float* __restrict__ S, int64_t h_in0, int64_t ho0, int64_t B) {
    constexpr int LANES = 32, CP = 64;
    __shared__ float4 ps[BAND2_SLOTS][4][9];
    __shared__ int32_t uo[BAND2_SLOTS][4];
    __shared__ __align__(16) float so[4][2][CP * 9];
    const int mi = threadIdx.x / LANES, cl = threadIdx.x % LANES;
    const int64_t mp0 = static_cast<int64_t>(blockIdx.x) * 4;
    const int64_t mp = mp0 + mi;
    const int64_t h = blockIdx.y;
    const int64_t hg = ho0 + h;
    const int h0 = band0[hg] - static_cast<int>(h_in0), nb = bandc[hg];
    const int64_t po = psi_off[hg];
    const int half = win / 2;
    const int nslot = nb * s;
    const int64_t C2 = C / 2;  // float4 per U bin row
    const int nt = static_cast<int>(nbo - mp0 < 4 ? nbo - mp0 : 4);
    for (int slot0 = 0; slot0 < nslot; slot0 += BAND2_SLOTS) {
        const int ns = min(BAND2_SLOTS, nslot - slot0);
        __syncthreads();
        for (int i = threadIdx.x; i < ns * 4; i += blockDim.x) {
            const int sl = i >> 2, t = i & 3;
            const int slot = slot0 + sl;
            const int bi = slot / s, q = slot - bi * s;
            const int64_t m = mp0 + t;
            const int kq = static_cast<int>(m) + wout * q;
            const bool fold = kq > half;
            const int idx = fold ? win - kq : kq;
            const float sg = fold ? -1.f : 1.f;
            const float2* src = psi_hat + ((po + bi) * nbi + idx) * K;
#pragma unroll
            for (int kk = 0; kk < 9; ++kk) {
                float2 v = make_float2(0.f, 0.f);
                if (m < nbo && kk < K) v = __ldg(src + kk);
                ps[sl][t][kk] = make_float4(v.x, v.y, sg * v.x, -sg * v.y);
            }
            uo[sl][t] = bi * static_cast<int>(nbi) + (m < nbo ? idx : 0);
        }
        __syncthreads();
        const bool mact = mp < nbo;
        for (int64_t b = 0; b < B; ++b) {
            for (int64_t c0 = 0; c0 < C; c0 += CP) {
                const int64_t c = c0 + 2 * cl;
                const int cn = static_cast<int>(C - c0 < CP ? C - c0 : CP);
                float2 re[9], im[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) re[k] = im[k] = make_float2(0.f, 0.f);
                if (mact && c < C) {
                    const float4* Ub = U + ((b * Hin + h0) * nbi * C + c) / 2;
                    constexpr int CH = 4;
                    float4 ua[CH], ub[CH];
                    auto load = [&](int sl0, float4 (&u)[CH]) {
#pragma unroll
                        for (int j = 0; j < CH; ++j) {
                            const int sl = sl0 + j;
                            u[j] = sl < ns ? __ldg(Ub + static_cast<int64_t>(uo[sl][mi]) * C2)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                    };
                    auto consume = [&](int sl0, const float4 (&u)[CH]) {
#pragma unroll
                        for (int j = 0; j < CH; ++j) {
                            if (sl0 + j >= ns) break;
                            const float4* pp = &ps[sl0 + j][mi][0];
                            const float2 UX = make_float2(u[j].x, u[j].y), UY = make_float2(u[j].z, u[j].w);
#pragma unroll
                            for (int k = 0; k < 9; ++k) {
                                const float4 qv = pp[k];
                                ffma2(re[k], qv.y, UY);
                                ffma2(re[k], qv.x, UX);
                                ffma2(im[k], qv.z, UY);
                                ffma2(im[k], qv.w, UX);
                            }
                        }
                    };
                    load(0, ua);
                    for (int sl0 = 0; sl0 < ns; sl0 += 2 * CH) {
                        if (sl0 + CH < ns) load(sl0 + CH, ub);
                        consume(sl0, ua);
                        if (sl0 + CH >= ns) break;
                        if (sl0 + 2 * CH < ns) load(sl0 + 2 * CH, ua);
                        consume(sl0 + CH, ub);
                    }
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    if (k < K) {
                        so[mi][0][(2 * cl) * K + k] = re[k].x;
                        so[mi][0][(2 * cl + 1) * K + k] = re[k].y;
                        so[mi][1][(2 * cl) * K + k] = im[k].x;
                        so[mi][1][(2 * cl + 1) * K + k] = im[k].y;
                    }
                __syncthreads();
                // contiguous rows of cn * K floats per (order, re/im), flattened over
                // (row, float4) so every pass keeps all threads busy
                const int rowlen = cn * K;
                const bool vec = (rowlen & 3) == 0 && (ldS & 3) == 0 && ((c0 * K) & 3) == 0;
                const int q4 = vec ? rowlen >> 2 : rowlen;
                float* sbase = S + (((b * Hout + h) * nbo + mp0) * 2) * ldS + c0 * K;
                for (int i = threadIdx.x; i < nt * 2 * q4; i += blockDim.x) {
                    const int r = i / q4, j = i - r * q4;
                    float* drow = sbase + static_cast<int64_t>(r) * ldS;
                    const float* srow = &so[r >> 1][r & 1][0];
                    if (vec) {
                        float4 v = reinterpret_cast<const float4*>(srow)[j];
                        float4* dst = reinterpret_cast<float4*>(drow) + j;
                        if (slot0 != 0) {
                            const float4 o = *dst;
                            v.x += o.x;
                            v.y += o.y;
                            v.z += o.z;
                            v.w += o.w;
                        }
                        *dst = v;
                    } else {
                        drow[j] = slot0 != 0 ? drow[j] + srow[j] : srow[j];
                    }
                }
            }
        }
    }
}

// Direct gather in the reference order (convolution.hpp:192-205), fp32:
// T[(b*Hout + h)*Wout + w][c*K + k] = sum_e vals[e][k] u[b][c][h_in][(w_rel + s w) % Win]
__global__ void __launch_bounds__(256) disco_gather_kernel(
    const float* __restrict__ x, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ h_in,
    const int32_t* __restrict__ w_rel, const float* __restrict__ vals, int64_t Hin, int64_t Win,
    int64_t Hout, int64_t Wout, int64_t stride, int K, int64_t C, int64_t ldS, float* __restrict__ T,
    int64_t h_in0, int64_t ho0) {
    const int64_t h = blockIdx.x, c = blockIdx.y, b = blockIdx.z;
    const float* u = x + (b * C + c) * Hin * Win - h_in0 * Win;  // global row index h_in[e]
    const int64_t e0 = row_ptr[ho0 + h], e1 = row_ptr[ho0 + h + 1];
    for (int64_t w = threadIdx.x; w < Wout; w += blockDim.x) {
        float acc[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[k] = 0.f;
        for (int64_t e = e0; e < e1; ++e) {
            int64_t col = w_rel[e] + stride * w;
            col %= Win;
            const float v = __ldg(u + static_cast<int64_t>(h_in[e]) * Win + col);
#pragma unroll
            for (int k = 0; k < 9; ++k)
                if (k < K) acc[k] = fmaf(__ldg(vals + e * K + k), v, acc[k]);
        }
        float* dst = T + ((b * Hout + h) * Wout + w) * ldS + c * K;
#pragma unroll
        for (int k = 0; k < 9; ++k)
            if (k < K) dst[k] = acc[k];
    }
}

// mix [cout][cin*K] -> transposed tf32 hi/lo table T[n = ci*K + k][co] (row stride ld)
__global__ void mix_t_split_kernel(const float* __restrict__ mix, int64_t cout, int64_t n, int64_t ld,
                                   float* __restrict__ hi, float* __restrict__ lo) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * ld) return;
    const int64_t r = i / ld, co = i % ld;
    const float x = co < cout ? mix[co * n + r] : 0.f;
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    const float h = __uint_as_float(u);
    hi[i] = h;
    lo[i] = x - h;
}

// Transpose band kernel (the adjoint of disco_band_kernel): for input row r and order m
// (< nbi), channel ci:
//   U'[b][r][m][ci] = sum_{h : r in band(h)} sum_k psi_t_hat_k[h, r](m) * S_k[b, h](m mod W_out)
// with S(m') for m' > W_out/2 taken as conj S(W_out - m') (Hermitian extension of the
// mixed output-ring spectra): zero-insertion upsampling by the stride replicates the
// spectrum, and the adjoint of the circular correlation is the circular convolution.
// A CTA owns RT consecutive input rows x 4 orders x 64 channels; it walks the output
// rows h whose band meets its row tile, loads S_k[b, h](m) (18 floats per thread) ONCE
// and scatters it into the tile rows of that band (RT complex accumulators per thread),
// so S is read once per (h, row tile) instead of once per (h, row): measured 20.1 ms at
// cfg3 B = 4 when each row re-read its S vectors.
constexpr int TB_RT = 16;
__global__ void __launch_bounds__(256) disco_band_t_kernel(
    const float* __restrict__ S, const float2* __restrict__ psi_t, const int32_t* __restrict__ band0,
    const int32_t* __restrict__ bandc, const int64_t* __restrict__ psi_off, const int32_t* __restrict__ tt_ptr,
    const int32_t* __restrict__ tt_h, int64_t Hin, int64_t nbi, int64_t Hout, int64_t nbo, int wout, int K,
    int64_t C, int64_t ldS, float2* __restrict__ Ut, int64_t B) {
    const int mi = threadIdx.x / 64, cl = threadIdx.x % 64;
    const int64_t m = static_cast<int64_t>(blockIdx.x) * 4 + mi;
    const int r0 = blockIdx.y * TB_RT;
    const int nr = min(TB_RT, static_cast<int>(Hin) - r0);
    if (m >= nbi) return;
    const int half = wout / 2;
    const int mo = static_cast<int>(m % wout);
    const bool cj = mo > half;
    const int mp = cj ? wout - mo : mo;
    const float sg = cj ? -1.f : 1.f;
    const int t0 = tt_ptr[blockIdx.y], t1 = tt_ptr[blockIdx.y + 1];
    for (int64_t b = 0; b < B; ++b) {
        const float* Sb = S + b * Hout * nbo * 2 * ldS;
        for (int64_t c0 = 0; c0 < C; c0 += 64) {
            const int64_t c = c0 + cl;
            if (c >= C) break;
            float2 acc[TB_RT];
#pragma unroll
            for (int i = 0; i < TB_RT; ++i) acc[i] = make_float2(0.f, 0.f);
            for (int t = t0; t < t1; ++t) {
                const int h = tt_h[t];
                const float* sr = Sb + (static_cast<int64_t>(h) * nbo + mp) * 2 * ldS + c * K;
                const float* si = sr + ldS;
                float xr[9], xi[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    xr[k] = k < K ? __ldg(sr + k) : 0.f;
                    xi[k] = k < K ? sg * __ldg(si + k) : 0.f;
                }
                const int bl = band0[h], bn = bandc[h];
                const int lo = max(bl, r0), hi = min(bl + bn, r0 + nr);
                const float2* pb = psi_t + (psi_off[h] + (lo - bl)) * nbi * K + m * K;
#pragma unroll
                for (int i = 0; i < TB_RT; ++i) {
                    const int r = r0 + i;
                    if (r < lo || r >= hi) continue;
                    const float2* pk = pb + static_cast<int64_t>(r - lo) * nbi * K;
                    float2 a = acc[i];
#pragma unroll
                    for (int k = 0; k < 9; ++k) {
                        if (k >= K) break;
                        const float2 p = __ldg(pk + k);
                        a.x = fmaf(p.x, xr[k], fmaf(-p.y, xi[k], a.x));
                        a.y = fmaf(p.x, xi[k], fmaf(p.y, xr[k], a.y));
                    }
                    acc[i] = a;
                }
            }
#pragma unroll
            for (int i = 0; i < TB_RT; ++i)
                if (i < nr) Ut[((b * Hin + r0 + i) * nbi + m) * C + c] = acc[i];
        }
    }
}

// Same contraction with the CTA's psi_t slice staged in shared memory once per CTA
// (reused over the batch and channel passes): the per-thread global psi loads of the
// kernel above (one LDG.64 per 4 FMA) made it load-bound (9.0 ms at cfg3 vs 1.8 ms for the
// forward band kernel, which stages psi the same way).  Dynamic SMEM psm[pair][4 orders][9]
// over the tile's (output row h, input row r) pairs in (h, r) order.
constexpr int TB_MAXH = 64;
__global__ void __launch_bounds__(256) disco_band_t2_kernel(
    const float* __restrict__ S, const float2* __restrict__ psi_t, const int32_t* __restrict__ band0,
    const int32_t* __restrict__ bandc, const int64_t* __restrict__ psi_off, const int32_t* __restrict__ tt_ptr,
    const int32_t* __restrict__ tt_h, int64_t Hin, int64_t nbi, int64_t Hout, int64_t nbo, int wout, int K,
    int64_t C, int64_t ldS, float2* __restrict__ Ut, int64_t B) {
    extern __shared__ float2 psm[];
    __shared__ int s_q0[TB_MAXH + 1], s_lo[TB_MAXH], s_hi[TB_MAXH];
    const int mi = threadIdx.x / 64, cl = threadIdx.x % 64;
    const int64_t mbase = static_cast<int64_t>(blockIdx.x) * 4;
    const int64_t m = mbase + mi;
    const int r0 = blockIdx.y * TB_RT;
    const int nr = min(TB_RT, static_cast<int>(Hin) - r0);
    const int t0 = tt_ptr[blockIdx.y], nt = tt_ptr[blockIdx.y + 1] - t0;
    if (threadIdx.x == 0) {
        int q = 0;
        for (int t = 0; t < nt; ++t) {
            const int h = tt_h[t0 + t];
            const int lo = max(band0[h], r0), hi = min(band0[h] + bandc[h], r0 + nr);
            s_q0[t] = q;
            s_lo[t] = lo;
            s_hi[t] = hi;
            q += max(0, hi - lo);
        }
        s_q0[nt] = q;
    }
    __syncthreads();
    const int nm = static_cast<int>(nbi - mbase < 4 ? nbi - mbase : 4);
    for (int t = 0; t < nt; ++t) {
        const int h = tt_h[t0 + t];
        const int lo = s_lo[t], n = s_hi[t] - lo;
        if (n <= 0) continue;
        // rows lo .. lo+n of h's band, orders mbase .. mbase+3, k < K: contiguous per row
        const float2* src = psi_t + (psi_off[h] + (lo - band0[h])) * nbi * K + mbase * K;
        for (int e = threadIdx.x; e < n * 4 * K; e += blockDim.x) {
            const int rr = e / (4 * K), rem = e - rr * 4 * K;
            const int mm = rem / K, k = rem - mm * K;
            psm[((s_q0[t] + rr) * 4 + mm) * 9 + k] =
                mm < nm ? __ldg(src + static_cast<int64_t>(rr) * nbi * K + rem) : make_float2(0.f, 0.f);
        }
    }
    __syncthreads();
    if (m >= nbi) return;
    const int half = wout / 2;
    const int mo = static_cast<int>(m % wout);
    const bool cj = mo > half;
    const int mp = cj ? wout - mo : mo;
    const float sg = cj ? -1.f : 1.f;
    for (int64_t b = 0; b < B; ++b) {
        const float* Sb = S + b * Hout * nbo * 2 * ldS;
        for (int64_t c0 = 0; c0 < C; c0 += 64) {
            const int64_t c = c0 + cl;
            if (c >= C) break;
            float2 acc[TB_RT];
#pragma unroll
            for (int i = 0; i < TB_RT; ++i) acc[i] = make_float2(0.f, 0.f);
            for (int t = 0; t < nt; ++t) {
                const int h = tt_h[t0 + t];
                const int lo = s_lo[t], hi = s_hi[t];
                if (hi <= lo) continue;
                const float* sr = Sb + (static_cast<int64_t>(h) * nbo + mp) * 2 * ldS + c * K;
                const float* si = sr + ldS;
                float xr[9], xi[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    xr[k] = k < K ? __ldg(sr + k) : 0.f;
                    xi[k] = k < K ? sg * __ldg(si + k) : 0.f;
                }
                const float2* pq = psm + (s_q0[t] - lo + r0) * 36 + mi * 9;  // pair of row r: pq + (r - r0) * 36
#pragma unroll
                for (int i = 0; i < TB_RT; ++i) {
                    const int r = r0 + i;
                    if (r < lo || r >= hi) continue;
                    const float2* pk = pq + i * 36;
                    float2 a = acc[i];
#pragma unroll
                    for (int k = 0; k < 9; ++k) {
                        if (k >= K) break;
                        const float2 p = pk[k];
                        a.x = fmaf(p.x, xr[k], fmaf(-p.y, xi[k], a.x));
                        a.y = fmaf(p.x, xi[k], fmaf(p.y, xr[k], a.y));
                    }
                    acc[i] = a;
                }
            }
#pragma unroll
            for (int i = 0; i < TB_RT; ++i)
                if (i < nr) Ut[((b * Hin + r0 + i) * nbi + m) * C + c] = acc[i];
        }
    }
}

// Even channel counts: disco_band_t2_kernel with a channel PAIR per thread accumulated in
// packed fp32x2 registers (FFMA2 with the staged psi value as the broadcast scalar): per
// (output row, input row) 9 broadcast LDS.64 feed 18 FFMA2 for two channels instead of
// 9 LDS + 36 FFMA for one.  The pair's 2 x 9 S values per re/im row are one contiguous
// 72-byte run, loaded as 9 LDG.64.  threads = 4 orders x 32 lanes, 64 channels per pass.
__global__ void __launch_bounds__(128, 4) disco_band_t3_kernel(
    const float* __restrict__ S, const float2* __restrict__ psi_t, const int32_t* __restrict__ band0,
    const int32_t* __restrict__ bandc, const int64_t* __restrict__ psi_off, const int32_t* __restrict__ tt_ptr,
    const int32_t* __restrict__ tt_h, int64_t Hin, int64_t nbi, int64_t Hout, int64_t nbo, int wout, int K,
    int64_t C, int64_t ldS, float2* __restrict__ Ut, int64_t B) {
    extern __shared__ float2 psm[];
    __shared__ int s_q0[TB_MAXH + 1], s_lo[TB_MAXH], s_hi[TB_MAXH];
    const int mi = threadIdx.x / 32, cl = threadIdx.x % 32;
    const int64_t mbase = static_cast<int64_t>(blockIdx.x) * 4;
    const int64_t m = mbase + mi;
    const int r0 = blockIdx.y * TB_RT;
    const int nr = min(TB_RT, static_cast<int>(Hin) - r0);
    const int t0 = tt_ptr[blockIdx.y], nt = tt_ptr[blockIdx.y + 1] - t0;
    if (threadIdx.x == 0) {
        int q = 0;
        for (int t = 0; t < nt; ++t) {
            const int h = tt_h[t0 + t];
            const int lo = max(band0[h], r0), hi = min(band0[h] + bandc[h], r0 + nr);
            s_q0[t] = q;
            s_lo[t] = lo;
            s_hi[t] = hi;
            q += max(0, hi - lo);
        }
        s_q0[nt] = q;
    }
    __syncthreads();
    const int nm = static_cast<int>(nbi - mbase < 4 ? nbi - mbase : 4);
    for (int t = 0; t < nt; ++t) {
        const int h = tt_h[t0 + t];
        const int lo = s_lo[t], n = s_hi[t] - lo;
        if (n <= 0) continue;
        const float2* src = psi_t + (psi_off[h] + (lo - band0[h])) * nbi * K + mbase * K;
        for (int e = threadIdx.x; e < n * 4 * K; e += blockDim.x) {
            const int rr = e / (4 * K), rem = e - rr * 4 * K;
            const int mm = rem / K, k = rem - mm * K;
            psm[((s_q0[t] + rr) * 4 + mm) * 9 + k] =
                mm < nm ? __ldg(src + static_cast<int64_t>(rr) * nbi * K + rem) : make_float2(0.f, 0.f);
        }
    }
    __syncthreads();
    if (m >= nbi) return;
    const int half = wout / 2;
    const int mo = static_cast<int>(m % wout);
    const bool cj = mo > half;
    const int mp = cj ? wout - mo : mo;
    const float sg = cj ? -1.f : 1.f;
    for (int64_t b = 0; b < B; ++b) {
        const float* Sb = S + b * Hout * nbo * 2 * ldS;
        for (int64_t c0 = 0; c0 < C; c0 += 64) {
            const int64_t c = c0 + 2 * cl;
            if (c >= C) break;
            // acc[i] = (re c, re c+1), acc[TB_RT + i] = (im c, im c+1) of input row r0 + i
            float2 are[TB_RT], aim[TB_RT];
#pragma unroll
            for (int i = 0; i < TB_RT; ++i) are[i] = aim[i] = make_float2(0.f, 0.f);
            for (int t = 0; t < nt; ++t) {
                const int h = tt_h[t0 + t];
                const int lo = s_lo[t], hi = s_hi[t];
                if (hi <= lo) continue;
                const float2* sr = reinterpret_cast<const float2*>(Sb + (static_cast<int64_t>(h) * nbo + mp) * 2 * ldS + c * 9);
                const float2* si = reinterpret_cast<const float2*>(reinterpret_cast<const float*>(sr) + ldS);
                float vr[18], vi[18];
#pragma unroll
                for (int j = 0; j < 9; ++j) {
                    const float2 a = __ldg(sr + j), bq = __ldg(si + j);
                    vr[2 * j] = a.x;
                    vr[2 * j + 1] = a.y;
                    vi[2 * j] = sg * bq.x;
                    vi[2 * j + 1] = sg * bq.y;
                }
                float2 xr[9], xi[9];  // (channel c, channel c+1) per basis function
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    xr[k] = make_float2(vr[k], vr[9 + k]);
                    xi[k] = make_float2(vi[k], vi[9 + k]);
                }
                const float2* pq = psm + (s_q0[t] - lo + r0) * 36 + mi * 9;
#pragma unroll
                for (int i = 0; i < TB_RT; ++i) {
                    const int r = r0 + i;
                    if (r < lo || r >= hi) continue;
                    const float2* pk = pq + i * 36;
                    float2 ar = are[i], ai = aim[i];
#pragma unroll
                    for (int k = 0; k < 9; ++k) {
                        const float2 p = pk[k];
                        // re += p.x xr - p.y xi,  im += p.x xi + p.y xr
                        ar = __ffma2_rn(make_float2(p.x, p.x), xr[k], ar);
                        ar = __ffma2_rn(make_float2(-p.y, -p.y), xi[k], ar);
                        ai = __ffma2_rn(make_float2(p.x, p.x), xi[k], ai);
                        ai = __ffma2_rn(make_float2(p.y, p.y), xr[k], ai);
                    }
                    are[i] = ar;
                    aim[i] = ai;
                }
            }
#pragma unroll
            for (int i = 0; i < TB_RT; ++i)
                if (i < nr)
                    *reinterpret_cast<float4*>(Ut + ((b * Hin + r0 + i) * nbi + m) * C + c) =
                        make_float4(are[i].x, aim[i].x, are[i].y, aim[i].y);
        }
    }
}

}  // namespace

void split_rows(const float* src, int64_t rows, int64_t cols, int64_t ld, float* hi, float* lo,
                cudaStream_t st) {
    const int64_t n = rows * ld;
    if (n == 0) return;
    split_rows_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(src, rows, cols, ld,
                                                                              hi, lo);
    SPH_LAUNCH_CHECK();
    count_launch();
}

void DiscoPlan::create(int in_kind_, int64_t in_nlat, int64_t in_nlon, int out_kind_,
                       int64_t out_nlat, int64_t out_nlon, int basis_kind, double cutoff,
                       int flags) {
    SPH_CUDA(cudaGetDevice(&device));
    in_kind = in_kind_;
    out_kind = out_kind_;
    hin = in_nlat;
    win = in_nlon;
    hout = out_nlat;
    wout = out_nlon;
    prec = flags & SPH_FLAG_PREC_MASK;
    require(prec <= SPH_PREC_FP32_SIMT, "disco plan: unknown precision mode");
    build_grid(in_kind, hin, win, in_colat, in_w);
    build_grid(out_kind, hout, wout, out_colat, out_w);
    const Basis basis = make_basis(basis_kind, cutoff);
    if (wout == 0 || win % wout != 0)  // convolution.hpp:143-145
        fail(SPH_ERR_INVALID_ARGUMENT,
             "assemble_disco: output longitudes must be a uniform subset of the input");
    require(hin < (1LL << 31) && win < (1LL << 31), "disco: grid too large");
    K = basis.n_real();
    require(K <= 9, "disco: at most 9 real basis functions supported");
    stride = win / wout;

    // ---- assemble (convolution.hpp:150-176), per output row in parallel
    std::vector<std::vector<int32_t>> rh(hout), rw(hout);
    std::vector<std::vector<double>> rv(hout), rb(hout);
    std::vector<double> lon(win);
    for (int64_t j = 0; j < win; ++j) lon[j] = 2.0 * kPi * static_cast<double>(j) / static_cast<double>(win);
    parallel_for(hout, [&](int64_t h) {
        const double theta_out = out_colat[h];
        for (int64_t hi = 0; hi < hin; ++hi) {
            const double theta_in = in_colat[hi];
            if (std::abs(theta_in - theta_out) >= basis.cutoff) continue;
            const double w_in = in_w[hi];
            for (int64_t wj = 0; wj < win; ++wj) {
                double dist, az;
                chart(theta_out, theta_in, lon[wj], dist, az);
                if (dist >= basis.cutoff) continue;
                rh[h].push_back(static_cast<int32_t>(hi));
                rw[h].push_back(static_cast<int32_t>(wj));
                for (int k = 0; k < K; ++k) {
                    const double bk = basis.eval_real(k, dist, az);
                    rv[h].push_back(bk * w_in);
                    rb[h].push_back(bk);
                }
            }
        }
    });
    row_ptr.assign(hout + 1, 0);
    for (int64_t h = 0; h < hout; ++h) {
        if (rh[h].empty())  // convolution.hpp:172-174
            fail(SPH_ERR_INVALID_ARGUMENT,
                 "assemble_disco: empty filter support (cutoff below grid spacing)");
        row_ptr[h + 1] = row_ptr[h] + static_cast<int64_t>(rh[h].size());
    }
    nnz = row_ptr[hout];
    h_in.resize(nnz);
    w_rel.resize(nnz);
    vals.resize(nnz * K);
    bases.resize(nnz * K);
    for (int64_t h = 0; h < hout; ++h) {
        std::copy(rh[h].begin(), rh[h].end(), h_in.begin() + row_ptr[h]);
        std::copy(rw[h].begin(), rw[h].end(), w_rel.begin() + row_ptr[h]);
        std::copy(rv[h].begin(), rv[h].end(), vals.begin() + row_ptr[h] * K);
        std::copy(rb[h].begin(), rb[h].end(), bases.begin() + row_ptr[h] * K);
    }
    upload(d_row_ptr, row_ptr);
    upload(d_h_in, h_in);
    upload(d_w_rel, w_rel);
    {
        std::vector<float> vf(vals.begin(), vals.end());
        upload(d_vals, vf);
    }

    // ---- longitude-Fourier tables
    nbi = win / 2 + 1;
    nbo = wout / 2 + 1;
    band0.assign(hout, 0);
    bandc.assign(hout, 0);
    psi_off.assign(hout + 1, 0);
    for (int64_t h = 0; h < hout; ++h) {
        int32_t lo = INT32_MAX, hi = -1;
        for (int64_t e = row_ptr[h]; e < row_ptr[h + 1]; ++e) {
            lo = std::min(lo, h_in[e]);
            hi = std::max(hi, h_in[e]);
        }
        band0[h] = lo;
        bandc[h] = hi - lo + 1;
        psi_off[h + 1] = psi_off[h] + bandc[h];
    }
    std::vector<double> cw(win), sw(win);
    for (int64_t j = 0; j < win; ++j) {
        const double a = -2.0 * kPi * static_cast<double>(j) / static_cast<double>(win);
        cw[j] = std::cos(a);
        sw[j] = std::sin(a);
    }
    const int64_t nrow = psi_off[hout];
    std::vector<float2> ph(static_cast<size_t>(nrow) * nbi * K);
    parallel_for(hout, [&](int64_t h) {
        std::vector<double> acc(static_cast<size_t>(bandc[h]) * nbi * K * 2, 0.0);
        for (int64_t e = row_ptr[h]; e < row_ptr[h + 1]; ++e) {
            const int64_t bi = h_in[e] - band0[h];
            const int64_t wr = w_rel[e];
            double* a = acc.data() + bi * nbi * K * 2;
            int64_t ph_idx = 0;  // (wr * m) mod win
            for (int64_t m = 0; m < nbi; ++m) {
                const double c = cw[ph_idx], s = sw[ph_idx];
                for (int k = 0; k < K; ++k) {
                    const double v = vals[e * K + k];
                    a[(m * K + k) * 2] += v * c;
                    a[(m * K + k) * 2 + 1] += v * s;
                }
                ph_idx += wr;
                if (ph_idx >= win) ph_idx -= win;
            }
        }
        float2* out = ph.data() + psi_off[h] * nbi * K;
        for (size_t i = 0; i < static_cast<size_t>(bandc[h]) * nbi * K; ++i)
            out[i] = make_float2(static_cast<float>(acc[2 * i]), static_cast<float>(acc[2 * i + 1]));
    });
    upload(d_psi_hat, ph);
    upload(d_band0, band0);
    upload(d_bandc, bandc);
    upload(d_psi_off, psi_off);
    fft_in.build(static_cast<int>(win));
    fft_out.build(static_cast<int>(wout));
}

namespace {
struct DiscoWs {
    int64_t ldS, u_off, s_off, y_off, whi_off, wlo_off, total;
};
// workspace for B samples, input rows nin, output rows nout
// The tensor core's fp32 accumulation loses precision linearly in the number of k-steps
// chained into one accumulator (measured at 360x720, 256 -> 256, random weights:
// relative error 1.6e-5 at c_in*K = 2304, 8.0e-6 at 1152, 4.0e-6 at 576, 2.1e-6 at 288,
// profiles/disco_ksplit_probe.py).  Mix reductions longer than kchunk run as chunk GEMMs
// over column slices of S and of the mix table, each writing its own partial spectrum;
// the C2R adds the partials in fp32 (round to nearest) while it loads them.
int64_t disco_kchunk() {
    static const int64_t kc = [] {
        const char* e = std::getenv("SPH_DISCO_KCHUNK");
        return e ? std::max<int64_t>(32, std::atoll(e) / 32 * 32) : int64_t{576};
    }();
    return kc;
}
int64_t disco_nchunks(const DiscoPlan& p, int64_t cin) {
    return p.prec == SPH_PREC_FP32_SIMT ? 1 : (cin * p.K + disco_kchunk() - 1) / disco_kchunk();
}

DiscoWs disco_ws(const DiscoPlan& p, int64_t B, int64_t cin, int64_t cout, int64_t nin, int64_t nout) {
    DiscoWs w;
    w.ldS = static_cast<int64_t>(round_up(cin * p.K, 4));
    const int64_t whi = cout * w.ldS * 4;
    int64_t o = 0;
    w.whi_off = o;
    o += round_up(whi, 256);
    w.wlo_off = o;
    o += round_up(whi, 256);
    if (p.prec == SPH_PREC_FP32_SIMT) {
        w.s_off = o;  // T (direct gather)
        o += round_up(B * nout * p.wout * w.ldS * 4, 256);
        w.u_off = w.y_off = 0;
    } else {
        w.u_off = o;
        o += round_up(B * nin * p.nbi * cin * 8, 256);
        w.s_off = o;
        o += round_up(B * nout * p.nbo * 2 * w.ldS * 4, 256);
        w.y_off = o;  // one partial spectrum per k chunk
        o += disco_nchunks(p, cin) * round_up(B * cout * nout * p.nbo * 2 * 4, 256);
    }
    w.total = o + 256;
    return w;
}
}  // namespace

int64_t DiscoPlan::workspace_bytes(int64_t B, int64_t cin, int64_t cout) const {
    return disco_ws(*this, B, cin, cout, hin, hout).total;
}

int64_t DiscoPlan::rows_workspace_bytes(int64_t B, int64_t cin, int64_t cout, int64_t nin,
                                        int64_t nout) const {
    return disco_ws(*this, B, cin, cout, nin, nout).total;
}

void DiscoPlan::input_rows(int64_t ho0, int64_t nout, int64_t* lo, int64_t* n) const {
    require(ho0 >= 0 && nout >= 1 && ho0 + nout <= hout, "disco: output row range");
    int64_t a = hin, b = -1;
    for (int64_t h = ho0; h < ho0 + nout; ++h) {
        a = std::min<int64_t>(a, band0[h]);
        b = std::max<int64_t>(b, band0[h] + bandc[h]);
    }
    *lo = a;
    *n = b - a;
}

bool DiscoPlan::pair_layout(int64_t cin) const {
    static const int band_mode = [] {
        const char* e = std::getenv("SPH_DISCO_BAND");
        return e ? std::atoi(e) : 2;
    }();
    return cin % 2 == 0 && band_mode == 2;
}

void DiscoPlan::apply(const float* x, const float* mix, int64_t B, int64_t cin, int64_t cout,
                      float* y, void* ws, cudaStream_t st) {
    apply_rows(x, 0, hin, 0, hout, mix, B, cin, cout, y, ws, st);
}

void DiscoPlan::apply_rows(const float* x, int64_t h_in0, int64_t nin, int64_t ho0, int64_t nout,
                           const float* mix, int64_t B, int64_t cin, int64_t cout, float* y,
                           void* ws, cudaStream_t st, const std::function<void(float2*)>* make_u) {
    require(B >= 0 && cin >= 1 && cout >= 1, "disco_apply: mix tensor shape mismatch");
    require(ho0 >= 0 && nout >= 1 && ho0 + nout <= hout, "disco_apply: output row range");
    require(h_in0 >= 0 && nin >= 1 && h_in0 + nin <= hin, "disco_apply: input row range");
    for (int64_t h = ho0; h < ho0 + nout; ++h)
        require(band0[h] >= h_in0 && band0[h] + bandc[h] <= h_in0 + nin,
                "disco_apply: input rows do not cover the filter support of the output rows");
    if (B == 0) return;
    DeviceGuard dguard(device);
    require_on_device(x, device, "disco_apply");
    require_on_device(y, device, "disco_apply");
    const DiscoWs w = disco_ws(*this, B, cin, cout, nin, nout);
    uint8_t* base = static_cast<uint8_t*>(ws);
    if (!base) {
        std::lock_guard<std::mutex> lk(mu);
        if (own_ws.n < static_cast<size_t>(w.total)) own_ws.alloc(w.total, true);
        base = own_ws.p;
    }
    float* whi = reinterpret_cast<float*>(base + w.whi_off);
    float* wlo = reinterpret_cast<float*>(base + w.wlo_off);
    split_rows(mix, cout, cin * K, w.ldS, whi, wlo, st);
    const bool direct = prec == SPH_PREC_FP32_SIMT;
    const int64_t rows_per_b = direct ? nout * wout : nout * nbo * 2;
    const int64_t kchunk = disco_kchunk();
    const int64_t Ktot = cin * K;
    const int64_t nchunks = direct ? 1 : disco_nchunks(*this, cin);
    auto make_gemm = [&](int64_t kc) {
        auto g = std::make_unique<GroupedGemm>();
        g->A = {nullptr, B * rows_per_b, kc, w.ldS};
        g->Bhi = {nullptr, cout, kc, w.ldS};
        g->Blo = {nullptr, cout, kc, w.ldS};
        g->store = STORE_TRANS;
        g->bn = cout >= 256 ? 256 : 128;
        static const int alo_mode = [] {
            const char* e = std::getenv("SPH_DISCO_ALO");
            return e ? std::atoi(e) : 1;
        }();
        if (alo_mode == 1 && prec != SPH_PREC_FP32_SIMT && cout <= 128) {
            // BK = 32 kernel: half the k-block rounds of the BK = 16 one at K = cin * 9
            // (decoder 64 -> 64: 4.26 -> 3.23 ms); with two N tiles (cout 256) the
            // BN = 256 BK = 16 kernel stays faster (1.42 vs 1.63 ms at cfg3)
            g->alo = true;
            g->bn = cout <= 64 ? 64 : 128;
        }
        // SPH_DISCO_MIX_BN=192: the CTA-pair bn = 192 kernel (A/B experiments)
        static const int mix_bn = std::getenv("SPH_DISCO_MIX_BN") ? std::atoi(std::getenv("SPH_DISCO_MIX_BN")) : 0;
        if (mix_bn == 192 && prec != SPH_PREC_FP32_SIMT) g->bn = 192;
        g->name = "gemm_disco_mix";
        // table multicast over 2 CTAs (cfg3: 1.386 ms vs 1.445 ms at the default 4)
        g->cluster = 2;
        require(B * rows_per_b < (1LL << 31), "disco: batch too large for one call");
        for (int64_t b = 0; b < B; ++b) {
            GemmGroup gr;
            gr.a_row0 = static_cast<int32_t>(b * rows_per_b);
            gr.b_row0 = 0;
            gr.M = static_cast<int32_t>(rows_per_b);
            gr.N = static_cast<int32_t>(cout);
            gr.K = static_cast<int32_t>(kc);
            gr.ldd = static_cast<int32_t>(rows_per_b);
            gr.zero_to = 0;
            gr.d_off = b * cout * rows_per_b;
            g->groups.push_back(gr);
        }
        g->finalize();
        return g;
    };
    const GroupedGemm* gp = nullptr;
    std::vector<std::pair<int64_t, const GroupedGemm*>> chunks;  // (k0, gemm)
    {
        std::lock_guard<std::mutex> lk(mu);
        if (nchunks <= 1) {
            auto& slot = gemm_cache[std::make_tuple(B, cin, cout, nout)];
            if (!slot) slot = make_gemm(Ktot);
            gp = slot.get();
        } else {
            for (int64_t k0 = 0; k0 < Ktot; k0 += kchunk) {
                const int64_t kc = std::min(kchunk, Ktot - k0);
                auto& slot = gemm_chunk_cache[std::make_tuple(B, cin, cout, nout, k0, kc)];
                if (!slot) slot = make_gemm(kc);
                chunks.emplace_back(k0, slot.get());
            }
        }
    }
    // D = A * mix^T; with a k split, chunk c writes partial spectrum c at D + c * dpart
    const int64_t dpart = static_cast<int64_t>(round_up(B * cout * nout * nbo * 2 * 4, 256)) / 4;
    auto run_mix = [&](const float* A, float* D) {
        if (chunks.empty()) {
            gemm_run(*gp, A, D, prec, st, whi, wlo);
            return;
        }
        for (size_t c = 0; c < chunks.size(); ++c) {
            const int64_t k0 = chunks[c].first;
            gemm_run(*chunks[c].second, A + k0, D + c * dpart, prec, st, whi + k0, wlo + k0);
        }
    };
    float* S = reinterpret_cast<float*>(base + w.s_off);
    if (direct) {
        dim3 grid(static_cast<unsigned>(nout), static_cast<unsigned>(cin), static_cast<unsigned>(B));
        require(cin <= 65535 && B <= 65535, "disco: too many channels for the gather grid");
        {
            ProfScope prof("disco_gather", st);
            disco_gather_kernel<<<grid, 256, 0, st>>>(x, d_row_ptr.p, d_h_in.p, d_w_rel.p, d_vals.p,
                                                      nin, win, nout, wout, stride, K, cin, w.ldS, S,
                                                      h_in0, ho0);
            SPH_LAUNCH_CHECK();
        }
        count_launch();
        run_mix(S, y);
        return;
    }
    float2* U = reinterpret_cast<float2*>(base + w.u_off);
    float* Yh = reinterpret_cast<float*>(base + w.y_off);
    if (make_u)
        (*make_u)(U);
    else
        fft_forward_cminor(fft_in, x, B, cin, nin, static_cast<int>(nbi), U, st, pair_layout(cin) ? 2 : 0);
    dim3 grid(static_cast<unsigned>((nbo + 3) / 4), static_cast<unsigned>(nout));
    require(nout <= 65535, "disco: grid too large");
    {
        // algorithmic bytes: U read once, S written once
        ProfScope prof("disco_band", st, 8.0 * B * nin * nbi * cin + 4.0 * B * nout * nbo * 2 * cin * K);
        if (pair_layout(cin))
            disco_band2_kernel<<<grid, 128, 0, st>>>(reinterpret_cast<const float4*>(U), d_psi_hat.p, d_band0.p,
                                                     d_bandc.p, d_psi_off.p, nin, nbi, nout, nbo,
                                                     static_cast<int>(win), static_cast<int>(wout),
                                                     static_cast<int>(stride), K, cin, w.ldS, S, h_in0, ho0, B);
        else
            disco_band_kernel<<<grid, 256, 0, st>>>(U, d_psi_hat.p, d_band0.p, d_bandc.p, d_psi_off.p, nin, nbi, nout,
                                                    nbo, static_cast<int>(win), static_cast<int>(wout),
                                                    static_cast<int>(stride), K, cin, w.ldS, S, h_in0, ho0, B);
        SPH_LAUNCH_CHECK();
    }
    count_launch();
    run_mix(S, Yh);
    fft_inverse_plain(fft_out, reinterpret_cast<const float2*>(Yh), B * cout * nout,
                      static_cast<int>(nbo), static_cast<float>(1.0 / static_cast<double>(win)), y,
                      st, static_cast<int>(std::max<int64_t>(1, static_cast<int64_t>(chunks.size()))), dpart / 2);
}

// ------------------------------------------------------------ transpose
void DiscoPlan::build_transpose() {
    std::lock_guard<std::mutex> lk(mu);
    if (t_ready) return;
    DeviceGuard dguard(device);
    // psi_t_hat with weights b_k * w_out[h] (convolution.hpp:251: scale = base * w_out)
    std::vector<double> cw(win), sw(win);
    for (int64_t j = 0; j < win; ++j) {
        const double a = -2.0 * kPi * static_cast<double>(j) / static_cast<double>(win);
        cw[j] = std::cos(a);
        sw[j] = std::sin(a);
    }
    const int64_t nrow = psi_off[hout];
    std::vector<float2> ph(static_cast<size_t>(nrow) * nbi * K);
    parallel_for(hout, [&](int64_t h) {
        std::vector<double> acc(static_cast<size_t>(bandc[h]) * nbi * K * 2, 0.0);
        const double wo = out_w[h];
        for (int64_t e = row_ptr[h]; e < row_ptr[h + 1]; ++e) {
            const int64_t bi = h_in[e] - band0[h];
            const int64_t wr = w_rel[e];
            double* a = acc.data() + bi * nbi * K * 2;
            int64_t ph_idx = 0;
            for (int64_t m = 0; m < nbi; ++m) {
                const double c = cw[ph_idx], s = sw[ph_idx];
                for (int k = 0; k < K; ++k) {
                    const double v = bases[e * K + k] * wo;
                    a[(m * K + k) * 2] += v * c;
                    a[(m * K + k) * 2 + 1] += v * s;
                }
                ph_idx += wr;
                if (ph_idx >= win) ph_idx -= win;
            }
        }
        float2* out = ph.data() + psi_off[h] * nbi * K;
        for (size_t i = 0; i < static_cast<size_t>(bandc[h]) * nbi * K; ++i)
            out[i] = make_float2(static_cast<float>(acc[2 * i]), static_cast<float>(acc[2 * i + 1]));
    });
    upload(d_psi_t, ph);
    // row-tile map: output rows h whose band meets input rows [TB_RT t, TB_RT (t+1))
    const int64_t ntile = (hin + TB_RT - 1) / TB_RT;
    std::vector<int32_t> ptr(ntile + 1, 0), hh;
    for (int64_t t = 0; t < ntile; ++t) {
        const int64_t r0 = t * TB_RT, r1 = std::min<int64_t>(hin, r0 + TB_RT);
        for (int64_t h = 0; h < hout; ++h)
            if (band0[h] < r1 && band0[h] + bandc[h] > r0) hh.push_back(static_cast<int32_t>(h));
        ptr[t + 1] = static_cast<int32_t>(hh.size());
    }
    upload(d_tb_ptr, ptr);
    upload(d_tb_h, hh);
    t_max_pairs = 0;
    t_max_h = 0;
    for (int64_t t = 0; t < ntile; ++t) {
        const int64_t r0 = t * TB_RT, r1 = std::min<int64_t>(hin, r0 + TB_RT);
        int64_t q = 0;
        for (int32_t i = ptr[t]; i < ptr[t + 1]; ++i) {
            const int64_t h = hh[i];
            q += std::max<int64_t>(0, std::min<int64_t>(band0[h] + bandc[h], r1) - std::max<int64_t>(band0[h], r0));
        }
        t_max_pairs = std::max(t_max_pairs, q);
        t_max_h = std::max<int64_t>(t_max_h, ptr[t + 1] - ptr[t]);
    }
    t_ready = true;
}

namespace {
struct DiscoTWs {
    int64_t ldc, ldS, v_off, s_off, u_off, thi_off, tlo_off, total;
};
DiscoTWs disco_t_ws(const DiscoPlan& p, int64_t B, int64_t cin, int64_t cout) {
    DiscoTWs w;
    w.ldc = static_cast<int64_t>(round_up(cout, 4));
    w.ldS = static_cast<int64_t>(round_up(cin * p.K, 4));
    int64_t o = 0;
    w.thi_off = o;
    o += round_up(cin * p.K * w.ldc * 4, 256);
    w.tlo_off = o;
    o += round_up(cin * p.K * w.ldc * 4, 256);
    w.v_off = o;  // planar V_hat [(b, h, m', re/im)][ldc]
    o += round_up(B * p.hout * p.nbo * 2 * w.ldc * 4, 256);
    w.s_off = o;  // mixed S [(b, h, m', re/im)][ldS]
    o += round_up(B * p.hout * p.nbo * 2 * w.ldS * 4, 256);
    w.u_off = o;  // U' [b][r][m][ci] complex
    o += round_up(B * p.hin * p.nbi * cin * 8, 256);
    w.total = o + 256;
    return w;
}
}  // namespace

int64_t DiscoPlan::transpose_workspace_bytes(int64_t B, int64_t cin, int64_t cout) const {
    return disco_t_ws(*this, B, cin, cout).total;
}

// convolution.hpp:226-266.  v_hat = channel-minor R2C of the output rings (planar re/im
// rows) -> mix^T GEMM (tcgen05 3xTF32, table mix^T [cin*K][cout]) -> transpose band
// kernel -> channel-minor C2R of the input rings (scale 1/W_in).
void DiscoPlan::transpose_apply(const float* v, const float* mix, int64_t B, int64_t cin, int64_t cout,
                                float* y, void* ws, cudaStream_t st) {
    require(cin >= 1 && cout >= 1 && B >= 0, "disco_transpose_apply: mix tensor shape mismatch");
    if (B == 0) return;
    build_transpose();
    DeviceGuard dguard(device);
    const DiscoTWs w = disco_t_ws(*this, B, cin, cout);
    uint8_t* base = static_cast<uint8_t*>(ws);
    if (!base) {
        std::lock_guard<std::mutex> lk(mu);
        if (own_ws.n < static_cast<size_t>(w.total)) own_ws.alloc(w.total, true);
        base = own_ws.p;
    }
    float* thi = reinterpret_cast<float*>(base + w.thi_off);
    float* tlo = reinterpret_cast<float*>(base + w.tlo_off);
    float* V = reinterpret_cast<float*>(base + w.v_off);
    float* S = reinterpret_cast<float*>(base + w.s_off);
    float2* Ut = reinterpret_cast<float2*>(base + w.u_off);
    const int64_t n = cin * K;
    {
        const int64_t tot = n * w.ldc;
        mix_t_split_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(mix, cout, n, w.ldc, thi,
                                                                                     tlo);
        SPH_LAUNCH_CHECK();
        count_launch();
    }
    // R2C of v's output rings, planar re/im rows: V[((b*hout + h)*nbo + m')*2 + ri][co]
    fft_forward_cminor(fft_out, v, B, cout, hout, static_cast<int>(nbo), reinterpret_cast<float2*>(V), st,
                       /*planar=*/true, w.ldc);
    const int64_t rows = B * hout * nbo * 2;
    const GroupedGemm* gp;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto& slot = gemm_t_cache[std::make_tuple(B, cin, cout)];
        if (!slot) {
            auto g = std::make_unique<GroupedGemm>();
            g->A = {nullptr, rows, cout, w.ldc};
            g->Bhi = {nullptr, n, cout, w.ldc};
            g->Blo = {nullptr, n, cout, w.ldc};
            g->store = STORE_ROW;
            // N = c_in * K: 576 at cfg3 is 3 x 192 (the bn = 256 tiling pads it to 768);
            // SPH_DISCO_MIXT_BN overrides
            static const int bn_env = std::getenv("SPH_DISCO_MIXT_BN") ? std::atoi(std::getenv("SPH_DISCO_MIXT_BN")) : 0;
            g->bn = bn_env == 128 || bn_env == 192 || bn_env == 256 ? bn_env
                    : n % 192 == 0 && n % 256 != 0     ? 192
                    : n >= 256                         ? 256
                                                       : 128;
            g->name = "gemm_disco_mix_t";
            require(rows < (1LL << 31), "disco_transpose_apply: batch too large for one call");
            GemmGroup gr;
            gr.a_row0 = 0;
            gr.b_row0 = 0;
            gr.M = static_cast<int32_t>(rows);
            gr.N = static_cast<int32_t>(n);
            gr.K = static_cast<int32_t>(cout);
            gr.ldd = static_cast<int32_t>(w.ldS);
            gr.zero_to = 0;
            gr.d_off = 0;
            g->groups.push_back(gr);
            g->finalize();
            slot = std::move(g);
        }
        gp = slot.get();
    }
    gemm_run(*gp, V, S, prec, st, thi, tlo);
    require(hin <= 65535, "disco_transpose_apply: grid too large");
    dim3 grid(static_cast<unsigned>((nbi + 3) / 4), static_cast<unsigned>((hin + TB_RT - 1) / TB_RT));
    {
        // algorithmic bytes: S read once, the input-grid spectrum written once
        ProfScope prof("disco_band_t", st, 4.0 * B * hout * nbo * 2 * cin * K + 8.0 * B * hin * nbi * cin);
        // psi_t staged per CTA when the tile's (h, r) pairs fit in shared memory
        const size_t psm_bytes = static_cast<size_t>(t_max_pairs) * 36 * sizeof(float2);
        if (t_max_h <= TB_MAXH && psm_bytes <= 200 * 1024) {
            static std::once_flag once;  // opt-in cap (the launch passes the actual size)
            std::call_once(once, [] {
                SPH_CUDA(cudaFuncSetAttribute(disco_band_t2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              200 * 1024));
            });
            static const bool t3 = !std::getenv("SPH_DISCO_T2");
            if (t3 && K == 9 && cin % 2 == 0 && w.ldS % 2 == 0) {
                // channel pairs + FFMA2 (the K = 9 Morlet basis; S rows of 2 x 9 floats per pair)
                static std::once_flag once3;
                std::call_once(once3, [] {
                    SPH_CUDA(cudaFuncSetAttribute(disco_band_t3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  200 * 1024));
                });
                disco_band_t3_kernel<<<grid, 128, psm_bytes, st>>>(S, d_psi_t.p, d_band0.p, d_bandc.p,
                                                                   d_psi_off.p, d_tb_ptr.p, d_tb_h.p, hin, nbi, hout,
                                                                   nbo, static_cast<int>(wout), K, cin, w.ldS, Ut, B);
            } else {
                disco_band_t2_kernel<<<grid, 256, psm_bytes, st>>>(S, d_psi_t.p, d_band0.p, d_bandc.p, d_psi_off.p,
                                                                   d_tb_ptr.p, d_tb_h.p, hin, nbi, hout, nbo,
                                                                   static_cast<int>(wout), K, cin, w.ldS, Ut, B);
            }
        } else {
            disco_band_t_kernel<<<grid, 256, 0, st>>>(S, d_psi_t.p, d_band0.p, d_bandc.p, d_psi_off.p, d_tb_ptr.p,
                                                      d_tb_h.p, hin, nbi, hout, nbo, static_cast<int>(wout), K, cin,
                                                      w.ldS, Ut, B);
        }
        SPH_LAUNCH_CHECK();
    }
    count_launch();
    fft_inverse_cminor(fft_in, Ut, B, cin, hin, static_cast<int>(nbi),
                       static_cast<float>(1.0 / static_cast<double>(win)), y, st);
}

}  // namespace sph
