// Longitude ring FFT kernels (see fft.cuh).  Conventions follow fft.hpp:85-86:
// forward sum_j x_j e^{-2 pi i jk/n}, inverse e^{+...}, no 1/n.
//
// Every kernel = IO.load (HBM -> shared, two real rings per complex ring) +
// transform + IO.store (shared -> HBM, with the real-pair split / parity fold).
// Transform engines, chosen per ring length by FftPlan::build:
//   * fft4      n = N1*45 (180, 360, 720, 1440): register-resident four-step
//               (fft4.cuh), 256 threads, 256/N1 complex rings per CTA
//   * stockham  other 2/3/5-smooth n: ping-pong shared-memory radix passes
//   * direct    anything else: O(n^2) DFT on a global scratch buffer
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <set>

#include "fft.cuh"
#include "gemm.cuh"  // EOI_TILE: the inverse GEMM's EOi field tiles
#include "fft4.cuh"

namespace sph {

namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_i(float2 a, float s) { return make_float2(-s * a.y, s * a.x); }

// ------------------------------------------------------------ Stockham engine
template <int R>
struct Dft {
    __device__ static void run(float2 (&v)[R], float s);
};
template <>
struct Dft<2> {
    __device__ static void run(float2 (&v)[2], float) {
        const float2 a = v[0];
        v[0] = cadd(a, v[1]);
        v[1] = csub(a, v[1]);
    }
};
template <>
struct Dft<3> {
    __device__ static void run(float2 (&v)[3], float s) {
        const float2 t = cadd(v[1], v[2]);
        const float2 d = csub(v[1], v[2]);
        const float2 m = make_float2(v[0].x - 0.5f * t.x, v[0].y - 0.5f * t.y);
        const float k = 0.86602540378443864676f;
        const float2 rd = mul_i(make_float2(k * d.x, k * d.y), s);
        v[0] = cadd(v[0], t);
        v[1] = cadd(m, rd);
        v[2] = csub(m, rd);
    }
};
template <>
struct Dft<4> {
    __device__ static void run(float2 (&v)[4], float s) {
        const float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
        const float2 t2 = cadd(v[1], v[3]), t3 = mul_i(csub(v[1], v[3]), s);
        v[0] = cadd(t0, t2);
        v[2] = csub(t0, t2);
        v[1] = cadd(t1, t3);
        v[3] = csub(t1, t3);
    }
};
template <>
struct Dft<5> {
    __device__ static void run(float2 (&v)[5], float s) {
        const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
        const float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
        const float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
        const float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
        const float2 p1 = make_float2(v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y);
        const float2 p2 = make_float2(v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y);
        const float2 q1 = mul_i(make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y), s);
        const float2 q2 = mul_i(make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y), s);
        v[0] = make_float2(v[0].x + a1.x + a2.x, v[0].y + a1.y + a2.y);
        v[1] = cadd(p1, q1);
        v[4] = csub(p1, q1);
        v[2] = cadd(p2, q2);
        v[3] = csub(p2, q2);
    }
};
template <>
struct Dft<8> {
    __device__ static void run(float2 (&v)[8], float s) {
        float2 e[4] = {v[0], v[2], v[4], v[6]};
        float2 o[4] = {v[1], v[3], v[5], v[7]};
        Dft<4>::run(e, s);
        Dft<4>::run(o, s);
        const float r = 0.70710678118654752440f;
        const float2 o1 = cmul(o[1], make_float2(r, s * r));
        const float2 o2 = mul_i(o[2], s);
        const float2 o3 = cmul(o[3], make_float2(-r, s * r));
        v[0] = cadd(e[0], o[0]);
        v[4] = csub(e[0], o[0]);
        v[1] = cadd(e[1], o1);
        v[5] = csub(e[1], o1);
        v[2] = cadd(e[2], o2);
        v[6] = csub(e[2], o2);
        v[3] = cadd(e[3], o3);
        v[7] = csub(e[3], o3);
    }
};

template <int R>
__device__ __forceinline__ void stockham_pass(const float2* __restrict__ src, float2* __restrict__ dst,
                                              int nrings, int n, int ns, const float2* tw, float s) {
    const int nb = n / R;
    const int total = nrings * nb;
    const int tstride = n / (ns * R);
    for (int b = threadIdx.x; b < total; b += FFT_THREADS) {
        const int ring = b / nb, j = b - ring * nb;
        const float2* sp = src + ring * n + j;
        const int k = j % ns;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float2 x = sp[r * nb];
            if (r > 0 && k > 0) {
                float2 w = __ldg(tw + k * r * tstride);
                if (s > 0) w.y = -w.y;
                x = cmul(x, w);
            }
            v[r] = x;
        }
        Dft<R>::run(v, s);
        float2* dp = dst + ring * n + (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dp[r * ns] = v[r];
    }
    __syncthreads();
}

struct FftArgs {
    int n, nstages;
    int radix[FFT_MAX_STAGES];
};

// returns the buffer holding the result
__device__ __forceinline__ float2* stockham(float2* a, float2* b, int nrings, const FftArgs& fa,
                                            const float2* tw, float s) {
    int ns = 1;
    for (int st = 0; st < fa.nstages; ++st) {
        switch (fa.radix[st]) {
            case 2: stockham_pass<2>(a, b, nrings, fa.n, ns, tw, s); break;
            case 3: stockham_pass<3>(a, b, nrings, fa.n, ns, tw, s); break;
            case 4: stockham_pass<4>(a, b, nrings, fa.n, ns, tw, s); break;
            case 5: stockham_pass<5>(a, b, nrings, fa.n, ns, tw, s); break;
            case 8: stockham_pass<8>(a, b, nrings, fa.n, ns, tw, s); break;
            default: break;
        }
        ns *= fa.radix[st];
        float2* t = a;
        a = b;
        b = t;
    }
    return a;
}

// ------------------------------------------------------------------- IO types
// Each IO maps blockIdx to P complex rings and provides load (HBM -> buf, ring-major)
// and store (buf, natural-order spectrum or signal -> HBM).

// forward SHT: ring pairs (ia, ib) of field f, folded rows r0.. -> E/O operand.
// P / n may be std::integral_constant (four-step path) so the index math folds.
// E/O layout (the forward Legendre GEMM's A operand), k-quad interleaved:
//   eo[((g * Rq + r / 4) * 2F + row) * 4 + r % 4],  g = 2 m + parity, row = 2 f + re/im,
//   Rq = Rp / 4 (ring pairs r in [R, Rp) hold zeros)
// i.e. per (g, quad) a [2F][4] block: a CTA of 4 ring pairs x FB fields writes FB*32-byte
// runs, and the GEMM loads [8 quads][128 rows][4] boxes (the SWIZZLE_NONE K-major
// core-matrix layout) with a 4D TMA map.  (The former [g][2F][Rp] layout gave 32-byte
// runs per CTA and a store phase of 1.56 of 2.86 ms at cfg2, SPH_FFT_DEBUG.)
struct FoldIO {
    int dbg;  // diagnostic (SPH_FFT_DEBUG): 1 skip store, 2 skip phase B + store, 4 loads only
    const float* x;
    const int2* rows;
    int R, nlat, mmax;
    float* eo;
    int64_t Rq, twoF;
    int fy_fast = 0;  // grid (field group, ring quad): concurrent CTAs fill adjacent E/O runs
    RingRows rrows{};  // optional per-latitude ring addressing (fft.cuh)
    // ring (field f, latitude row) of x
    __device__ __forceinline__ const float* ring(int64_t f, int row, int n) const {
        return rrows.roff ? x + f * rrows.fstr[row] + rrows.roff[row] : x + (f * nlat + row) * static_cast<int64_t>(n);
    }
    __device__ __forceinline__ int qx_of() const { return fy_fast ? blockIdx.y : blockIdx.x; }
    __device__ __forceinline__ int fy_of() const { return fy_fast ? blockIdx.x : blockIdx.y; }
    // slot p of a CTA -> (ring pair, field); false if outside [0, R) x [0, F).
    // P % 4 == 0 (all fast paths): 4 ring pairs x P/4 fields per CTA; otherwise P ring
    // pairs of one field (small fallback transforms)
    template <class PT>
    __device__ __forceinline__ bool slot(PT P, int p, int& r, int& f) const {
        const int np = static_cast<int>(P);
        if (np % 4 == 0) {
            r = 4 * qx_of() + (p & 3);
            f = (np / 4) * fy_of() + (p >> 2);
        } else {
            r = np * blockIdx.x + p;
            f = blockIdx.y;
        }
        return r < R && f < twoF / 2;
    }
    // slot p's ring pair (a, b) for the fused direct-load kernel
    template <class PT>
    __device__ __forceinline__ bool rings(PT P, int n, int p, const float*& pa, const float*& pb,
                                          float& sb) const {
        int rr, f;
        if (!slot(P, p, rr, f)) return false;
        const int2 rw = rows[rr];
        pa = ring(f, rw.x, n);
        pb = ring(f, rw.y < 0 ? rw.x : rw.y, n);
        sb = rw.y < 0 ? 0.f : 1.f;
        return true;
    }
    template <class PT, class NT>
    __device__ __forceinline__ void load(float2* buf, PT P, NT n, int ld) const {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        if ((n & 3) == 0) {
            const int n4 = n / 4;
            for (int j = warp; j < P; j += nw) {  // one ring pair per warp
                float4* d = reinterpret_cast<float4*>(buf + j * ld);
                int rr, f;
                if (slot(P, j, rr, f)) {
                    const int2 rw = rows[rr];
                    const float4* pa = reinterpret_cast<const float4*>(ring(f, rw.x, n));
                    const float4* pb = reinterpret_cast<const float4*>(ring(f, rw.y < 0 ? rw.x : rw.y, n));
                    const bool hb = rw.y >= 0;
                    for (int k4 = lane; k4 < n4; k4 += 32) {
                        const float4 va = __ldg(pa + k4);
                        float4 vb = __ldg(pb + k4);
                        if (!hb) vb = make_float4(0.f, 0.f, 0.f, 0.f);
                        d[2 * k4] = make_float4(va.x, vb.x, va.y, vb.y);
                        d[2 * k4 + 1] = make_float4(va.z, vb.z, va.w, vb.w);
                    }
                } else {
                    for (int k4 = lane; k4 < n4; k4 += 32) {
                        d[2 * k4] = make_float4(0.f, 0.f, 0.f, 0.f);
                        d[2 * k4 + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
            }
        } else {
            for (int j = warp; j < P; j += nw) {
                int rr, f;
                const bool ok = slot(P, j, rr, f);
                const int2 rw = ok ? rows[rr] : make_int2(0, -1);
                const float* xa = ok ? ring(f, rw.x, n) : x;
                const float* xb = ok && rw.y >= 0 ? ring(f, rw.y, n) : x;
                for (int k = lane; k < n; k += 32) {
                    float2 v = make_float2(0.f, 0.f);
                    if (ok) {
                        v.x = xa[k];
                        if (rw.y >= 0) v.y = xb[k];
                    }
                    buf[j * ld + k] = v;
                }
            }
        }
    }
    // store: thread (m, row rr of the 2*FB rows [f re, f im, ...]) writes the E and O
    // float4 of the CTA's 4 ring pairs; the 2*FB lanes of one m cover a contiguous
    // FB*32-byte run of the quad-interleaved layout
    template <class PT, class NT>
    __device__ __forceinline__ void store(const float2* buf, PT P, NT n, int ld) const {
        const int64_t gstride = Rq * twoF * 4;  // floats per (m, parity) group
        if (static_cast<int>(P) % 4 != 0) {     // fallback: scalar stores, slot j -> pair
            const int np = static_cast<int>(P);
            for (int i = threadIdx.x; i < np * mmax; i += blockDim.x) {
                const int j = i % np, m = i / np;
                int r, f;
                if (!slot(P, j, r, f)) continue;
                const float2* zr = buf + j * ld;
                const float2 z = zr[m];
                const float2 zc = zr[m == 0 ? 0 : static_cast<int>(n) - m];
                const float ar = 0.5f * (z.x + zc.x), ai = 0.5f * (z.y - zc.y);
                const float br = 0.5f * (z.y + zc.y), bi = -0.5f * (z.x - zc.x);
                float* em = eo + (2 * static_cast<int64_t>(m)) * gstride +
                            ((static_cast<int64_t>(r / 4)) * twoF + 2 * f) * 4 + (r & 3);
                em[0] = ar + br;
                em[4] = ai + bi;
                em[gstride] = ar - br;
                em[gstride + 4] = ai - bi;
            }
            return;
        }
        store_job(buf, P, n, ld, qx_of(), fy_of());
    }
    // quad path for the job (quad qx, field group fy)
    template <class PT, class NT>
    __device__ __forceinline__ void store_job(const float2* buf, PT P, NT n, int ld, int qx, int fy) const {
        const int64_t gstride = Rq * twoF * 4;
        const int FB = static_cast<int>(P) / 4, NR = 2 * FB;
        const int rr = threadIdx.x % NR;
        const int mstep = blockDim.x / NR;
        const int fl = rr >> 1, ri = rr & 1;
        const int64_t row = 2 * static_cast<int64_t>(FB * fy + fl) + ri;
        if (row >= twoF) return;
        float* base = eo + (static_cast<int64_t>(qx) * twoF + row) * 4;
        for (int m = threadIdx.x / NR; m < mmax; m += mstep) {
            float e[4], o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2* zr = buf + (4 * fl + j) * ld;
                const float2 z = zr[m];
                const float2 zc = zr[m == 0 ? 0 : static_cast<int>(n) - m];
                const float ar = 0.5f * (z.x + zc.x), ai = 0.5f * (z.y - zc.y);
                const float br = 0.5f * (z.y + zc.y), bi = -0.5f * (z.x - zc.x);
                e[j] = ri ? ai + bi : ar + br;
                o[j] = ri ? ai - bi : ar - br;
            }
            float* em = base + (2 * static_cast<int64_t>(m)) * gstride;
            *reinterpret_cast<float4*>(em) = make_float4(e[0], e[1], e[2], e[3]);
            *reinterpret_cast<float4*>(em + gstride) = make_float4(o[0], o[1], o[2], o[3]);
        }
    }
};

// inverse SHT: Ev/Od -> Hermitian spectra of the ring pair -> rings.  Input layout
// EOi[r][t][g][32] (t = 32-row field tile, g = 2 m + parity, rows 2f + re/im), written by
// the inverse GEMM's TMA-store epilogue (GroupedGemm::d_mode 1) in 128-byte pieces, so
// a CTA of one folded row r and P = 8 fields reads 64-byte halves of one contiguous
// chunk (the neighbouring CTA reads the other halves).  (The former [m][parity][R][2F]
// layout gave 64-byte runs ~6 MB apart: the load phase alone took 1.56 of 2.4 ms at
// cfg2, SPH_FFT_DEBUG.)
struct UnfoldIO {
    int dbg;  // diagnostic (SPH_FFT_DEBUG, bits << 4): 16 skip stores, 32 loads only
    const float* eoi;
    const int2* rows;
    int R, nlat, msynth, lmax;
    int64_t F, twoF;
    float* y;
    int64_t T;  // EOI_TILE-row field tiles (gemm.cuh)
    RingRows rrows{};  // optional per-latitude ring addressing (fft.cuh)
    __device__ __forceinline__ float* ring(int64_t f, int row, int n) const {
        return rrows.roff ? y + f * rrows.fstr[row] + rrows.roff[row] : y + (f * nlat + row) * static_cast<int64_t>(n);
    }
    template <int N1, int N2>
    __device__ __forceinline__ void store_b(int P, int N, int p, int k1, const float2 (&b)[N2]) const {
        const int64_t f = static_cast<int64_t>(blockIdx.x) * P + p;
        if (dbg & 16) {
            if (b[0].x == 12345.f) y[0] = b[N2 - 1].y;  // keep phase B live
            return;
        }
        if (f >= F) return;
        const int2 rw = rows[blockIdx.y];
        float* pa = ring(f, rw.x, N) + k1;
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) pa[N1 * k2] = b[k2].x;
        if (rw.y >= 0) {
            float* pb = ring(f, rw.y, N) + k1;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) pb[N1 * k2] = b[k2].y;
        }
    }
    template <class PT, class NT>
    __device__ __forceinline__ void load(float2* buf, PT P, NT n, int ld) const {
        const int r = blockIdx.y;  // field tiles fastest: neighbouring CTAs read adjacent runs
        const int64_t f0 = static_cast<int64_t>(blockIdx.x) * P;
        const int nf = static_cast<int>(min(static_cast<int64_t>(P), F - f0));
        const int j = threadIdx.x % P;
        const int mstep = blockDim.x / P;
        const int m0 = threadIdx.x / P;
        float2* zr = buf + j * ld;
        for (int k = msynth + m0; k <= n - msynth; k += mstep) zr[k] = make_float2(0.f, 0.f);
        if (j >= nf) {
            for (int m = m0; m < msynth; m += mstep) {
                zr[m] = make_float2(0.f, 0.f);
                if (m) zr[n - m] = make_float2(0.f, 0.f);
            }
            return;
        }
        const bool pair = rows[r].y >= 0;
        const int64_t row = 2 * (f0 + j);  // re row of field f0 + j
        const float2* e = reinterpret_cast<const float2*>(
            eoi + ((static_cast<int64_t>(r) * T + row / EOI_TILE) * 2 * msynth) * EOI_TILE + (row % EOI_TILE));
        const int64_t so = EOI_TILE / 2;  // parity stride in float2 (next g)
        const int64_t sm = EOI_TILE;      // order stride in float2 (g += 2)
        // batches of UB orders: all 2*UB loads issued before any use (memory-level
        // parallelism for the latency-bound load phase)
        constexpr int UB = 8;
        for (int mb = m0; mb < msynth; mb += UB * mstep) {
            float2 ev[UB], od[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int m = mb + u * mstep;
                const bool ok = m < msynth;
                const float2* em = e + (ok ? m : 0) * sm;
                ev[u] = (ok && (lmax - m + 1) / 2 > 0) ? __ldg(em) : make_float2(0.f, 0.f);
                od[u] = (ok && (lmax - m) / 2 > 0) ? __ldg(em + so) : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int m = mb + u * mstep;
                if (m >= msynth) break;
                const float2 ha = cadd(ev[u], od[u]);
                const float2 hb = pair ? csub(ev[u], od[u]) : make_float2(0.f, 0.f);
                if (m == 0) {
                    zr[0] = make_float2(ha.x, hb.x);  // Im of the DC bin is dropped
                } else {
                    zr[m] = make_float2(ha.x - hb.y, ha.y + hb.x);      // ha + i hb
                    zr[n - m] = make_float2(ha.x + hb.y, hb.x - ha.y);  // conj ha + i conj hb
                }
            }
        }
    }
    template <class PT, class NT>
    __device__ __forceinline__ void store(const float2* buf, PT P, NT n, int ld) const {
        const int r = blockIdx.y;  // field tiles fastest: neighbouring CTAs read adjacent runs
        const int64_t f0 = static_cast<int64_t>(blockIdx.x) * P;
        const int nf = static_cast<int>(min(static_cast<int64_t>(P), F - f0));
        const int2 rw = rows[r];
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int j = warp; j < nf; j += nw) {
            const float2* zr = buf + j * ld;
            float* pa = ring(f0 + j, rw.x, n);
            float* pb = rw.y >= 0 ? ring(f0 + j, rw.y, n) : pa;
            for (int k = lane; k < n; k += 32) {
                pa[k] = zr[k].x;
                if (rw.y >= 0) pb[k] = zr[k].y;
            }
        }
    }
};

// plain forward: rings [nrings][n] -> bins [nrings][nbins] * scale (distsim.hpp:413-430)
struct PlainFwdIO {
    const float* rings;
    int64_t nrings;
    int nbins;
    float scale;
    float2* bins;
    template <class PT, class NT>
    __device__ __forceinline__ void load(float2* buf, PT P, NT n, int ld) const {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * P;
        for (int i = threadIdx.x; i < P * n; i += blockDim.x) {
            const int j = i / n, k = i - j * n;
            const int64_t ra = 2 * (c0 + j), rb = ra + 1;
            buf[j * ld + k] = make_float2(ra < nrings ? rings[ra * n + k] : 0.f,
                                          rb < nrings ? rings[rb * n + k] : 0.f);
        }
    }
    template <class PT, class NT>
    __device__ __forceinline__ void store(const float2* buf, PT P, NT n, int ld) const {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * P;
        for (int o = threadIdx.x; o < P * 2 * nbins; o += blockDim.x) {
            const int m = o % nbins;
            const int jj = o / nbins;
            const int j = jj >> 1, which = jj & 1;
            const int64_t ring = 2 * (c0 + j) + which;
            if (ring >= nrings) continue;
            const float2 z = buf[j * ld + m];
            const float2 zc = buf[j * ld + (m == 0 ? 0 : n - m)];
            const float2 v = which ? make_float2(0.5f * (z.y + zc.y), -0.5f * (z.x - zc.x))
                                   : make_float2(0.5f * (z.x + zc.x), 0.5f * (z.y - zc.y));
            bins[ring * nbins + m] = make_float2(v.x * scale, v.y * scale);
        }
    }
};

// plain inverse: half spectra [nrings][nbins] -> rings [nrings][n] * scale
// Hermitian half-spectrum load into the complex ring buffer of a C2R pair (z = A + iB):
// element i of the P x (n/2+1) block is (slot j, bin k) = at(i) with spectra ha (ring A),
// hb (ring B).  Batches of 4 elements per thread issue all their global loads before
// any shared-memory store (one load pair in flight per thread was latency-bound: 62 %
// long-scoreboard stalls at the DISCO C2R).
template <class PT, class NT, class At, class Get>
__device__ __forceinline__ void load_half_spectra(float2* buf, PT P, NT n, int ld, At at, Get get) {
    constexpr int U = 4;
    const int half = n / 2, nh = half + 1;
    const int total = P * nh;
    for (int i0 = threadIdx.x; i0 < total; i0 += U * blockDim.x) {
        float2 ha[U], hb[U];
        int jj[U], kk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            jj[u] = -1;
            ha[u] = hb[u] = make_float2(0.f, 0.f);
            if (i < total) {
                at(i, jj[u], kk[u]);
                get(jj[u], kk[u], ha[u], hb[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (jj[u] < 0) continue;
            const int j = jj[u], k = kk[u];
            float2 a = ha[u], b = hb[u];
            if (k == 0 || 2 * k == n) { a.y = 0.f; b.y = 0.f; }
            buf[j * ld + k] = make_float2(a.x - b.y, a.y + b.x);
            if (k != 0 && 2 * k != n) buf[j * ld + n - k] = make_float2(a.x + b.y, b.x - a.y);
        }
    }
}

struct PlainInvIO {
    static constexpr bool kRegStore = true;  // fft4_unfold_kernel (register stores)
    const float2* bins;
    int64_t nrings;
    int nbins;
    float scale;
    float* rings;
    int dbg = 0;
    int nparts = 1;            // partial spectra summed on load (DISCO k split)
    int64_t part_stride = 0;   // float2 between partials
    template <int N1, int N2>
    __device__ __forceinline__ void store_b(int P, int n, int p, int k1, const float2 (&b)[N2]) const {
        const int64_t ra = 2 * (static_cast<int64_t>(blockIdx.x) * P + p), rb = ra + 1;
        if (ra < nrings) {
            float* d = rings + ra * n + k1;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) d[N1 * k2] = b[k2].x * scale;
        }
        if (rb < nrings) {
            float* d = rings + rb * n + k1;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) d[N1 * k2] = b[k2].y * scale;
        }
    }
    // each half-spectrum bin k <= n/2 is loaded once and written at k and n - k
    template <class PT, class NT>
    __device__ __forceinline__ void load(float2* buf, PT P, NT n, int ld) const {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * P;
        const int nh = n / 2 + 1;
        load_half_spectra(
            buf, P, n, ld, [&](int i, int& j, int& k) { j = i / nh; k = i - j * nh; },
            [&](int j, int k, float2& ha, float2& hb) {
                const int64_t ra = 2 * (c0 + j), rb = ra + 1;
                if (k < nbins) {
                    if (ra < nrings) ha = __ldg(bins + ra * nbins + k);
                    if (rb < nrings) hb = __ldg(bins + rb * nbins + k);
                    for (int q = 1; q < nparts; ++q) {  // k-split partial spectra, fp32 sum
                        const float2* bq = bins + q * part_stride;
                        if (ra < nrings) ha = cadd(ha, __ldg(bq + ra * nbins + k));
                        if (rb < nrings) hb = cadd(hb, __ldg(bq + rb * nbins + k));
                    }
                }
            });
    }
    template <class PT, class NT>
    __device__ __forceinline__ void store(const float2* buf, PT P, NT n, int ld) const {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * P;
        for (int i = threadIdx.x; i < P * 2 * n; i += blockDim.x) {
            const int jj = i / n, k = i - jj * n;
            const int j = jj >> 1, which = jj & 1;
            const int64_t ring = 2 * (c0 + j) + which;
            if (ring >= nrings) continue;
            const float2 z = buf[j * ld + k];
            rings[ring * n + k] = (which ? z.y : z.x) * scale;
        }
    }
};

// channel-minor forward (DISCO input): block (c-tile of 2P channels, row hi, batch b).
// planar = 0: U[b][hi][m][c] complex; planar = 1 (DISCO transpose): real planes
// U[((b*H + hi)*nbins + m)*2 + re/im][c] so a GEMM can take re and im rows with K = c;
// planar = 2 (DISCO band, even C): per bin, channel pairs as (re c, re c+1, im c, im c+1).
struct CminorIO {
    const float* x;
    int64_t C, H;
    int nbins;
    float2* U;
    int planar;
    int64_t ldp;  // planar row stride (floats, >= C)
    int dbg = 0;
    // slot p = channels (c0 + 2p, c0 + 2p + 1) of row hi, batch b (fused direct-load kernel)
    template <class PT>
    __device__ __forceinline__ bool rings(PT P, int n, int p, const float*& pa, const float*& pb,
                                          float& sb) const {
        const int64_t ca = static_cast<int64_t>(blockIdx.x) * 2 * P + 2 * p, cb = ca + 1;
        const int64_t hi = blockIdx.y, b = blockIdx.z;
        if (ca >= C) return false;
        pa = x + ((b * C + ca) * H + hi) * n;
        pb = cb < C ? x + ((b * C + cb) * H + hi) * n : pa;
        sb = cb < C ? 1.f : 0.f;
        return true;
    }
    template <class PT, class NT>
    __device__ __forceinline__ void load(float2* buf, PT P, NT n, int ld) const {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 2 * P;
        const int64_t hi = blockIdx.y, b = blockIdx.z;
        for (int i = threadIdx.x; i < P * n; i += blockDim.x) {
            const int j = i / n, k = i - j * n;
            const int64_t ca = c0 + 2 * j, cb = ca + 1;
            buf[j * ld + k] = make_float2(ca < C ? x[((b * C + ca) * H + hi) * n + k] : 0.f,
                                 cb < C ? x[((b * C + cb) * H + hi) * n + k] : 0.f);
        }
    }
    template <class PT, class NT>
    __device__ __forceinline__ void store(const float2* buf, PT P, NT n, int ld) const {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 2 * P;
        const int64_t hi = blockIdx.y, b = blockIdx.z;
        float2* Ub = U + (b * H + hi) * static_cast<int64_t>(nbins) * C;
        float* Up = reinterpret_cast<float*>(U) + (b * H + hi) * static_cast<int64_t>(nbins) * 2 * ldp;
        if (planar == 2) {
            // channel-pair interleaved (re c, re c+1, im c, im c+1): one thread per (bin,
            // pair) forms both channels from the pair's complex ring and stores one float4
            // (C even, so a pair never straddles the channel range)
            for (int o = threadIdx.x; o < nbins * P; o += blockDim.x) {
                const int j = o % P;
                const int m = o / P;
                if (c0 + 2 * j >= C) continue;
                const float2 z = buf[j * ld + m];
                const float2 zc = buf[j * ld + (m == 0 ? 0 : n - m)];
                const float4 v = make_float4(0.5f * (z.x + zc.x), 0.5f * (z.y + zc.y), 0.5f * (z.y - zc.y),
                                             -0.5f * (z.x - zc.x));
                reinterpret_cast<float4*>(Ub)[(static_cast<int64_t>(m) * C + c0 + 2 * j) >> 1] = v;
            }
            return;
        }
        for (int o = threadIdx.x; o < nbins * 2 * P; o += blockDim.x) {
            const int cl = o % (2 * P);
            const int m = o / (2 * P);
            if (c0 + cl >= C) continue;
            const int j = cl >> 1;
            const float2 z = buf[j * ld + m];
            const float2 zc = buf[j * ld + (m == 0 ? 0 : n - m)];
            const float2 v = (cl & 1) ? make_float2(0.5f * (z.y + zc.y), -0.5f * (z.x - zc.x))
                                      : make_float2(0.5f * (z.x + zc.x), 0.5f * (z.y - zc.y));
            if (planar == 2) {
                // channel-pair interleaved: (re c, re c+1, im c, im c+1) per even c
                const int64_t cc = c0 + cl;
                float* pu = reinterpret_cast<float*>(Ub) + (static_cast<int64_t>(m) * C + (cc & ~1LL)) * 2 + (cc & 1);
                pu[0] = v.x;
                pu[2] = v.y;
            } else if (planar) {
                float* pm = Up + static_cast<int64_t>(m) * 2 * ldp + c0 + cl;
                pm[0] = v.x;
                pm[ldp] = v.y;
            } else {
                Ub[static_cast<int64_t>(m) * C + c0 + cl] = v;
            }
        }
    }
};

// channel-minor inverse (DISCO transpose output): half spectra V[b][hi][m][c] (m < nbins)
// -> rings y[b][c][hi][0..n) * scale; block (c-tile of 2P channels, row hi, batch b), two
// channels per complex ring (z = A + iB), Im of DC / Nyquist dropped (real synthesis)
struct CminorInvIO {
    static constexpr bool kRegStore = true;  // fft4_unfold_kernel (register stores)
    const float2* V;
    int64_t C, H;
    int nbins;
    float scale;
    float* y;
    int dbg = 0;
    template <int N1, int N2>
    __device__ __forceinline__ void store_b(int P, int n, int p, int k1, const float2 (&b)[N2]) const {
        const int64_t ca = static_cast<int64_t>(blockIdx.x) * 2 * P + 2 * p, cb = ca + 1;
        const int64_t hi = blockIdx.y, bb = blockIdx.z;
        if (ca < C) {
            float* d = y + ((bb * C + ca) * H + hi) * n + k1;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) d[N1 * k2] = b[k2].x * scale;
        }
        if (cb < C) {
            float* d = y + ((bb * C + cb) * H + hi) * n + k1;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) d[N1 * k2] = b[k2].y * scale;
        }
    }
    template <class PT, class NT>
    __device__ __forceinline__ void load(float2* buf, PT P, NT n, int ld) const {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 2 * P;
        const int64_t hi = blockIdx.y, b = blockIdx.z;
        const float2* Vb = V + (b * H + hi) * static_cast<int64_t>(nbins) * C;
        // channel pairs fastest (coalesced channel-minor reads), each bin loaded once
        load_half_spectra(
            buf, P, n, ld, [&](int i, int& j, int& k) { j = i % P; k = i / P; },
            [&](int j, int k, float2& ha, float2& hb) {
                const int64_t ca = c0 + 2 * j, cb = ca + 1;
                if (k < nbins) {
                    if (ca < C) ha = __ldg(Vb + static_cast<int64_t>(k) * C + ca);
                    if (cb < C) hb = __ldg(Vb + static_cast<int64_t>(k) * C + cb);
                }
            });
    }
    template <class PT, class NT>
    __device__ __forceinline__ void store(const float2* buf, PT P, NT n, int ld) const {
        const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 2 * P;
        const int64_t hi = blockIdx.y, b = blockIdx.z;
        for (int i = threadIdx.x; i < P * n; i += blockDim.x) {
            const int j = i / n, k = i - j * n;
            const int64_t ca = c0 + 2 * j, cb = ca + 1;
            const float2 z = buf[j * ld + k];
            if (ca < C) y[((b * C + ca) * H + hi) * n + k] = z.x * scale;
            if (cb < C) y[((b * C + cb) * H + hi) * n + k] = z.y * scale;
        }
    }
};

// ------------------------------------------------------------------- kernels
template <int N1, bool INV, class IO>
__global__ void __launch_bounds__(fft4::THREADS, 2) fft4_kernel(IO io, const float2* __restrict__ twT) {
    extern __shared__ float2 sm4[];
    constexpr int N = N1 * 45, P = fft4::THREADS / N1, LD = N + 2;  // padded ring stride
    using PC = std::integral_constant<int, P>;
    using NC = std::integral_constant<int, N>;
    io.load(sm4, PC{}, NC{}, LD);
    __syncthreads();
    fft4::transform<N1, 45, LD, INV>(sm4, twT);
    io.store(sm4, PC{}, NC{}, LD);
}


// Forward SHT ring transform, fused IO (n = N1*45): phase A loads its N1 strided ring
// samples of both rings of the pair straight from HBM into registers (a warp reads 32
// consecutive samples per load -> 128-byte segments, 2*N1 independent loads in flight
// per thread), so the input never takes a shared-memory staging pass.
// FOLD_THREADS = 256 (8 ring slots = 4 ring pairs x 2 fields at N1 = 32, 2 CTAs / SM).
// Measured at cfg2: 512 threads (16 slots, 128-byte E/O runs, 1 CTA / SM) 2.42 ms vs
// 2.30 ms -- the store phase (~1.0 ms) is not run-length bound; the load / compute /
// store phases of a CTA serialise (SPH_FFT_DEBUG: loads 0.69, +A+B 1.27 ms).  A
// persistent 1-CTA/SM variant that bulk-copied the next job's rings into a staging
// buffer during phase B / stores measured 2.50 ms (8 warps per SM for the compute
// phases cost more than the overlap gained).
constexpr int FOLD_THREADS = 256;
// Generic over IO (FoldIO: ring pairs of the SHT; CminorIO: channel pairs of a DISCO
// input row): IO::rings(P, n, p, pa, pb, sb) gives the two real rings of slot p.
template <int N1, class IO, int T = FOLD_THREADS>
__global__ void __launch_bounds__(T, 512 / T) fft4_fold_kernel(IO io, const float2* __restrict__ twT) {
    extern __shared__ float2 smf[];
    constexpr int N2 = 45, N = N1 * N2, P = T / N1, LD = N + 2;
    for (int it = threadIdx.x; it < P * N2; it += T) {
        const int p = it / N2, n2 = it - p * N2;
        float2 a[N1];
        const float *pa, *pb;
        float sb;
        if (io.rings(std::integral_constant<int, P>{}, N, p, pa, pb, sb)) {
            pa += n2;
            pb += n2;
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) a[n1] = make_float2(__ldg(pa + N2 * n1), sb * __ldg(pb + N2 * n1));
        } else {
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) a[n1] = make_float2(0.f, 0.f);
        }
        if (io.dbg & 4) {
            float2* r = smf + p * LD + n2;
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) r[N2 * k1] = a[k1];
        } else {
            fft4::phase_a_store<N1, N2, LD, false>(a, smf, p, n2, twT);
        }
    }
    __syncthreads();
    if (io.dbg & 6) return;
    float2 b[N2];
    fft4::phase_b_regs<N1, N2, LD, false>(smf, b);
    __syncthreads();
    {
        const int p = threadIdx.x / N1, k1 = threadIdx.x - p * N1;
        float2* dst = smf + p * LD + k1;
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) dst[N1 * k2] = b[k2];
    }
    __syncthreads();
    if (io.dbg & 1) return;
    io.store(smf, std::integral_constant<int, P>{}, std::integral_constant<int, N>{}, LD);
}

// Inverse SHT ring transform, fused IO: phase B stores the synthesised ring samples
// straight from registers to HBM (Re -> ring a, Im -> ring b; a warp writes 32
// consecutive samples per store).
// Generic over IO (UnfoldIO, PlainInvIO, CminorInvIO): IO::load builds the spectra in
// shared memory, IO::store_b(P, N1, p, k1, b) writes thread (p, k1)'s N2 outputs
// X[k1 + N1 k2] of ring slot p straight from registers (coalesced over k1).
template <int N1, class IO, int T = fft4::THREADS>
__global__ void __launch_bounds__(T, 512 / T) fft4_unfold_kernel(IO io, const float2* __restrict__ twT) {
    extern __shared__ float2 smu[];
    constexpr int N2 = 45, N = N1 * N2, P = T / N1, LD = N + 2;
    io.load(smu, std::integral_constant<int, P>{}, std::integral_constant<int, N>{}, LD);
    __syncthreads();
    if (io.dbg & 32) return;
    for (int it = threadIdx.x; it < P * N2; it += T) {
        const int p = it / N2, n2 = it - p * N2;
        float2 a[N1];
        const float2* r = smu + p * LD + n2;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) a[n1] = r[N2 * n1];
        fft4::phase_a_store<N1, N2, LD, true>(a, smu, p, n2, twT);
    }
    __syncthreads();
    float2 b[N2];
    fft4::phase_b_regs<N1, N2, LD, true>(smu, b);
    const int p = threadIdx.x / N1, k1 = threadIdx.x - p * N1;
    io.template store_b<N1, N2>(P, N, p, k1, b);
}

template <bool INV, class IO>
__global__ void __launch_bounds__(FFT_THREADS) stockham_kernel(IO io, FftArgs a, const float2* __restrict__ tw,
                                                               int rpb) {
    extern __shared__ float2 sms[];
    float2* b0 = sms;
    float2* b1 = sms + static_cast<size_t>(rpb) * a.n;
    io.load(b0, rpb, a.n, a.n);
    __syncthreads();
    float2* res = stockham(b0, b1, rpb, a, tw, INV ? 1.f : -1.f);
    io.store(res, rpb, a.n, a.n);
}

// direct fallback: one CTA per complex ring, O(n^2), scratch in global memory
template <bool INV, class IO>
__global__ void direct_kernel(IO io, const float2* __restrict__ tw, int n, float2* __restrict__ scratch) {
    const size_t blk = blockIdx.x + static_cast<size_t>(gridDim.x) * (blockIdx.y + static_cast<size_t>(gridDim.y) * blockIdx.z);
    float2* in = scratch + blk * 2 * n;
    float2* out = in + n;
    io.load(in, 1, n, n);
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        float2 acc = make_float2(0.f, 0.f);
        for (int j = 0; j < n; ++j) {
            float2 w = __ldg(tw + static_cast<int64_t>(j) * k % n);
            if (INV) w.y = -w.y;
            acc = cadd(acc, cmul(in[j], w));
        }
        out[k] = acc;
    }
    __syncthreads();
    io.store(out, 1, n, n);
}

FftArgs make_args(const FftPlan& fp) {
    FftArgs a;
    a.n = fp.n;
    a.nstages = fp.nstages;
    for (int i = 0; i < FFT_MAX_STAGES; ++i) a.radix[i] = fp.radix[i];
    return a;
}

template <class K>
void set_smem_once(K kernel, size_t bytes) {
    static std::mutex mu;
    static std::set<const void*> done;
    const void* key = reinterpret_cast<const void*>(kernel);
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert(key).second)
        SPH_CUDA(cudaFuncSetAttribute(key, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(bytes)));
}

template <class T, class = void>
struct has_regstore : std::false_type {};
template <class T>
struct has_regstore<T, std::void_t<decltype(T::kRegStore)>> : std::true_type {};

template <int N1, bool INV, class IO>
void launch4(const FftPlan& fp, const IO& io, dim3 grid, cudaStream_t st) {
    const size_t sm = static_cast<size_t>(fft4::THREADS / N1) * (N1 * 45 + 2) * sizeof(float2);
    if constexpr (INV && has_regstore<IO>::value) {
        // inverse transforms whose IO can store phase B's registers directly (one shared
        // memory pass fewer than fft4_kernel)
        set_smem_once(fft4_unfold_kernel<N1, IO>, sm);
        fft4_unfold_kernel<N1, IO><<<grid, fft4::THREADS, sm, st>>>(io, fp.twT.p);
        return;
    }
    set_smem_once(fft4_kernel<N1, INV, IO>, sm);
    fft4_kernel<N1, INV, IO><<<grid, fft4::THREADS, sm, st>>>(io, fp.twT.p);
}

// CTA size of the fused SHT ring transforms (SPH_FFT_FOLD_THREADS / SPH_FFT_UNFOLD_THREADS,
// 128 or 256)
int fold_threads() {
    static const int t = std::getenv("SPH_FFT_FOLD_THREADS") ? std::atoi(std::getenv("SPH_FFT_FOLD_THREADS")) : FOLD_THREADS;
    return t == 128 ? 128 : 256;
}
int unfold_threads() {
    static const int t = std::getenv("SPH_FFT_UNFOLD_THREADS") ? std::atoi(std::getenv("SPH_FFT_UNFOLD_THREADS")) : fft4::THREADS;
    return t == 128 ? 128 : 256;
}

template <bool FWD>
void launch_fused(const FftPlan& fp, const FoldIO& fio, const UnfoldIO& uio, dim3 grid, cudaStream_t st) {
    const int T = FWD ? fold_threads() : unfold_threads();
    auto go = [&](auto n1c) {
        constexpr int N1 = decltype(n1c)::value;
        const size_t sm = static_cast<size_t>(T / N1) * (N1 * 45 + 2) * sizeof(float2);
        auto run = [&](auto tc) {
            constexpr int TT = decltype(tc)::value;
            if constexpr (TT / N1 >= 4) {  // FoldIO's quad path needs 4 ring pairs per CTA
                if (FWD) {
                    set_smem_once(fft4_fold_kernel<N1, FoldIO, TT>, sm);
                    fft4_fold_kernel<N1, FoldIO, TT><<<grid, TT, sm, st>>>(fio, fp.twT.p);
                } else {
                    set_smem_once(fft4_unfold_kernel<N1, UnfoldIO, TT>, sm);
                    fft4_unfold_kernel<N1, UnfoldIO, TT><<<grid, TT, sm, st>>>(uio, fp.twT.p);
                }
            } else {
                fail(SPH_ERR_RUNTIME, "fft4: CTA too small for the ring split");
            }
        };
        if (T == 128) run(std::integral_constant<int, 128>{});
        else run(std::integral_constant<int, 256>{});
    };
    switch (fp.fft4_n1) {
        case 4: go(std::integral_constant<int, 4>{}); break;
        case 8: go(std::integral_constant<int, 8>{}); break;
        case 16: go(std::integral_constant<int, 16>{}); break;
        case 32: go(std::integral_constant<int, 32>{}); break;
        default: fail(SPH_ERR_RUNTIME, "fft4: unsupported split");
    }
    SPH_LAUNCH_CHECK();
    count_launch();
}

// rows-per-block of the engine chosen for this plan
int rpb_of(const FftPlan& fp) {
    return fp.fft4_n1 ? fft4::THREADS / fp.fft4_n1 : fp.direct ? 1 : fp.rows_per_block;
}

template <bool INV, class IO>
void run_transform(const FftPlan& fp, const IO& io, dim3 grid, cudaStream_t st, const char* name,
                   double bytes) {
    ProfScope prof(name, st, bytes);
    if (fp.fft4_n1) {
        switch (fp.fft4_n1) {
            case 4: launch4<4, INV>(fp, io, grid, st); break;
            case 8: launch4<8, INV>(fp, io, grid, st); break;
            case 16: launch4<16, INV>(fp, io, grid, st); break;
            case 32: launch4<32, INV>(fp, io, grid, st); break;
            default: fail(SPH_ERR_RUNTIME, "fft4: unsupported split");
        }
    } else if (!fp.direct) {
        const size_t sm = static_cast<size_t>(fp.n) * sizeof(float2) * 2 * fp.rows_per_block;
        set_smem_once(stockham_kernel<INV, IO>, 200 * 1024);
        stockham_kernel<INV, IO><<<grid, FFT_THREADS, sm, st>>>(io, make_args(fp), fp.tw.p, fp.rows_per_block);
    } else {
        const size_t nblk = static_cast<size_t>(grid.x) * grid.y * grid.z;
        DevBuf<float2> scratch(nblk * 2 * fp.n, false);
        direct_kernel<INV, IO><<<grid, 256, 0, st>>>(io, fp.tw.p, fp.n, scratch.p);
        SPH_LAUNCH_CHECK();
        SPH_CUDA(cudaStreamSynchronize(st));  // scratch lifetime
    }
    SPH_LAUNCH_CHECK();
    count_launch();
}

}  // namespace

void FftPlan::build(int n_) {
    n = n_;
    require(n >= 1, "fft: length must be >= 1");
    nstages = 0;
    direct = false;
    fft4_n1 = 0;
    int m = n;
    while (m % 8 == 0 && m != 1) { radix[nstages++] = 8; m /= 8; }
    while (m % 4 == 0) { radix[nstages++] = 4; m /= 4; }
    while (m % 2 == 0) { radix[nstages++] = 2; m /= 2; }
    for (int p : {3, 5})
        while (m % p == 0) { radix[nstages++] = p; m /= p; }
    if (m != 1 || nstages > FFT_MAX_STAGES) direct = true;
    if (n % 45 == 0 && (n / 45 == 4 || n / 45 == 8 || n / 45 == 16 || n / 45 == 32)) fft4_n1 = n / 45;
    std::vector<float2> h(n);
    for (int q = 0; q < n; ++q) {
        const double ang = -2.0 * M_PI * static_cast<double>(q) / static_cast<double>(n);
        h[q] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
    }
    tw.alloc(n, false);
    SPH_CUDA(cudaMemcpy(tw.p, h.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
    if (fft4_n1) {  // twT[k1*45 + n2] = W_n^{n2 k1}
        std::vector<float2> t(n);
        for (int k1 = 0; k1 < fft4_n1; ++k1)
            for (int n2 = 0; n2 < 45; ++n2) {
                const double ang = -2.0 * M_PI * static_cast<double>(n2 * k1) / static_cast<double>(n);
                t[k1 * 45 + n2] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
            }
        twT.alloc(n, false);
        SPH_CUDA(cudaMemcpy(twT.p, t.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
    }
    // stockham: complex rings per CTA so that the ping-pong buffers fit ~110 KB
    int rpb = 16;
    while (rpb > 1 && static_cast<size_t>(n) * sizeof(float2) * 2 * rpb > 110 * 1024) --rpb;
    rows_per_block = rpb;
    if (!direct && static_cast<size_t>(n) * sizeof(float2) * 2 * rows_per_block > 200 * 1024) direct = true;
}

void fft_forward_fold(const FftPlan& fp, const FoldRows& fr, const float* x, int64_t F, int nlat,
                      int mmax, float* eo, int64_t ld_eo, cudaStream_t st, RingRows rr) {
    if (F == 0) return;
    require(F <= 65535, "fft: at most 65535 fields per call");
    const int P = fp.fft4_n1 ? fold_threads() / fp.fft4_n1 : rpb_of(fp);
    static const int fft_dbg = std::getenv("SPH_FFT_DEBUG") ? std::atoi(std::getenv("SPH_FFT_DEBUG")) : 0;
    require(ld_eo % 4 == 0, "fft: E/O ring-pair padding must be a multiple of 4");
    FoldIO io{fft_dbg, x, fr.d_rows.p, fr.R, nlat, mmax, eo, ld_eo / 4, 2 * F};
    io.rrows = rr;
    // field groups fastest (measured at cfg2: 2.21 -> 2.11 ms): concurrently running CTAs
    // write adjacent 64-byte runs of the same (m, parity, quad) E/O row instead of runs
    // 32 KB apart; SPH_FFT_FY_FAST=0 restores quad-fastest
    static const int fy_fast = std::getenv("SPH_FFT_FY_FAST") ? std::atoi(std::getenv("SPH_FFT_FY_FAST")) : 1;
    dim3 grid;
    if (P % 4 == 0) {
        const int64_t FB = P / 4;
        io.fy_fast = fy_fast;
        grid = fy_fast ? dim3(static_cast<unsigned>((F + FB - 1) / FB), (fr.R + 3) / 4)
                       : dim3((fr.R + 3) / 4, static_cast<unsigned>((F + FB - 1) / FB));
    } else {  // fallback transforms write pairs < R only: zero the [R, Rp) padding first
        grid = dim3((fr.R + P - 1) / P, static_cast<unsigned>(F));
        if (fr.R % 4 != 0)
            SPH_CUDA(cudaMemsetAsync(eo, 0, sizeof(float) * 2 * F * ld_eo * 2 * mmax, st));
    }
    const double bytes = 4.0 * F * (static_cast<double>(nlat) * fp.n + 4.0 * mmax * fr.R);
    if (fp.fft4_n1) {
        ProfScope prof("fft_fwd_fold", st, bytes);
        launch_fused<true>(fp, io, UnfoldIO{}, grid, st);
        return;
    }
    run_transform<false>(fp, io, grid, st, "fft_fwd_fold", bytes);
}

void fft_inverse_unfold(const FftPlan& fp, const FoldRows& fr, const float* eoi, int64_t F,
                        int nlat, int mmax, int msynth, int lmax, int64_t ld_eo, float* y,
                        cudaStream_t st, RingRows rr) {
    (void)mmax;
    if (F == 0) return;
    require(F <= 65535, "fft: at most 65535 fields per call");
    const int P = fp.fft4_n1 ? unfold_threads() / fp.fft4_n1 : rpb_of(fp);
    (void)ld_eo;  // EOi is [m][parity][R][2F] (transposed GEMM store)
    static const int fft_dbg = std::getenv("SPH_FFT_DEBUG") ? std::atoi(std::getenv("SPH_FFT_DEBUG")) : 0;
    UnfoldIO io{fft_dbg, eoi, fr.d_rows.p, fr.R, nlat, msynth, lmax, F, 2 * F, y, (2 * F + EOI_TILE - 1) / EOI_TILE};
    io.rrows = rr;
    require(fr.R <= 65535, "fft: too many latitude rows");
    dim3 grid(static_cast<unsigned>((F + P - 1) / P), static_cast<unsigned>(fr.R));
    const double bytes = 4.0 * F * (static_cast<double>(nlat) * fp.n + 4.0 * msynth * fr.R);
    if (fp.fft4_n1) {
        ProfScope prof("fft_inv_unfold", st, bytes);
        launch_fused<false>(fp, FoldIO{}, io, grid, st);
        return;
    }
    run_transform<true>(fp, io, grid, st, "fft_inv_unfold", bytes);
}

void fft_forward_plain(const FftPlan& fp, const float* rings, int64_t nrings, int nbins,
                       float scale, float2* bins, cudaStream_t st) {
    if (nrings == 0) return;
    const int P = rpb_of(fp);
    const int64_t nc = (nrings + 1) / 2;
    const int64_t nblk = (nc + P - 1) / P;
    require(nblk < (1LL << 31), "fft: too many rings");
    PlainFwdIO io{rings, nrings, nbins, scale, bins};
    run_transform<false>(fp, io, dim3(static_cast<unsigned>(nblk)), st, "fft_fwd_plain",
                         4.0 * nrings * (fp.n + 2.0 * nbins));
}

void fft_inverse_plain(const FftPlan& fp, const float2* bins, int64_t nrings, int nbins,
                       float scale, float* rings, cudaStream_t st, int nparts, int64_t part_stride) {
    if (nrings == 0) return;
    const int P = rpb_of(fp);
    const int64_t nc = (nrings + 1) / 2;
    const int64_t nblk = (nc + P - 1) / P;
    require(nblk < (1LL << 31), "fft: too many rings");
    PlainInvIO io{bins, nrings, nbins, scale, rings};
    io.nparts = std::max(1, nparts);
    io.part_stride = part_stride;
    run_transform<true>(fp, io, dim3(static_cast<unsigned>(nblk)), st, "fft_inv_plain",
                        4.0 * nrings * (fp.n + 2.0 * io.nparts * nbins));
}

void fft_forward_cminor(const FftPlan& fp, const float* x, int64_t B, int64_t C, int64_t H,
                        int nbins, float2* U, cudaStream_t st, int planar, int64_t ldp) {
    if (B * C * H == 0) return;
    require(planar != 2 || C % 2 == 0, "disco fft: pair-interleaved layout needs an even channel count");
    require(H <= 65535 && B <= 65535, "disco fft: too many rows");
    const int P = rpb_of(fp);
    CminorIO io{x, C, H, nbins, U, planar, ldp > 0 ? ldp : C};
    dim3 grid(static_cast<unsigned>((C + 2 * P - 1) / (2 * P)), static_cast<unsigned>(H),
              static_cast<unsigned>(B));
    if (fp.fft4_n1 && FOLD_THREADS == fft4::THREADS) {
        // fused: phase A loads its strided ring samples straight from HBM into registers
        // (the generic kernel staged the rings through shared memory first)
        ProfScope prof("fft_fwd_cminor", st, 4.0 * B * C * H * (fp.n + 2.0 * nbins));
        auto go = [&](auto n1c) {
            constexpr int N1 = decltype(n1c)::value;
            const size_t smf = static_cast<size_t>(FOLD_THREADS / N1) * (N1 * 45 + 2) * sizeof(float2);
            set_smem_once(fft4_fold_kernel<N1, CminorIO>, smf);
            fft4_fold_kernel<N1, CminorIO><<<grid, FOLD_THREADS, smf, st>>>(io, fp.twT.p);
        };
        switch (fp.fft4_n1) {
            case 4: go(std::integral_constant<int, 4>{}); break;
            case 8: go(std::integral_constant<int, 8>{}); break;
            case 16: go(std::integral_constant<int, 16>{}); break;
            default: go(std::integral_constant<int, 32>{}); break;
        }
        SPH_LAUNCH_CHECK();
        count_launch();
        return;
    }
    run_transform<false>(fp, io, grid, st, "fft_fwd_cminor", 4.0 * B * C * H * (fp.n + 2.0 * nbins));
}

void fft_inverse_cminor(const FftPlan& fp, const float2* V, int64_t B, int64_t C, int64_t H, int nbins,
                        float scale, float* y, cudaStream_t st) {
    if (B * C * H == 0) return;
    require(H <= 65535 && B <= 65535, "disco fft: too many rows");
    const int P = rpb_of(fp);
    CminorInvIO io{V, C, H, nbins, scale, y};
    dim3 grid(static_cast<unsigned>((C + 2 * P - 1) / (2 * P)), static_cast<unsigned>(H),
              static_cast<unsigned>(B));
    run_transform<true>(fp, io, grid, st, "fft_inv_cminor", 4.0 * B * C * H * (fp.n + 2.0 * nbins));
}

}  // namespace sph
