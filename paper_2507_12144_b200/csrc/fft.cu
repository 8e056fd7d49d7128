// Longitude ring FFT kernels (see fft.cuh).  Conventions follow fft.hpp:85-86:
// forward sum_j x_j e^{-2 pi i jk/n}, inverse e^{+...}, no 1/n.
#include <cmath>

#include "fft.cuh"

namespace sph {

namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse): s = -1 / +1
__device__ __forceinline__ float2 mul_i(float2 a, float s) { return make_float2(-s * a.y, s * a.x); }

// Small DFTs in registers; s = -1 forward, +1 inverse (twiddle sign).
template <int R>
struct Dft {
    // generic prime radix via the n-point twiddle table (W_R^q = W_n^{q n/R})
    __device__ static void run(float2 (&v)[R], const float2* tw, int n, float s) {
        float2 out[R];
        const int step = n / R;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            float2 acc = v[0];
#pragma unroll
            for (int r = 1; r < R; ++r) {
                float2 w = tw[((r * k) % R) * step];
                if (s > 0) w.y = -w.y;
                acc = cadd(acc, cmul(v[r], w));
            }
            out[k] = acc;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = out[k];
    }
};
template <>
struct Dft<2> {
    __device__ static void run(float2 (&v)[2], const float2*, int, float) {
        const float2 a = v[0];
        v[0] = cadd(a, v[1]);
        v[1] = csub(a, v[1]);
    }
};
template <>
struct Dft<3> {
    __device__ static void run(float2 (&v)[3], const float2*, int, float s) {
        const float2 t = cadd(v[1], v[2]);
        const float2 d = csub(v[1], v[2]);
        const float2 m = make_float2(v[0].x - 0.5f * t.x, v[0].y - 0.5f * t.y);
        const float k = 0.86602540378443864676f;  // sin(2 pi / 3)
        const float2 rd = mul_i(make_float2(k * d.x, k * d.y), s);  // s*i*k*d
        v[0] = cadd(v[0], t);
        v[1] = cadd(m, rd);
        v[2] = csub(m, rd);
    }
};
template <>
struct Dft<4> {
    __device__ static void run(float2 (&v)[4], const float2*, int, float s) {
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
    __device__ static void run(float2 (&v)[5], const float2*, int, float s) {
        const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
        const float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
        const float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
        const float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
        const float2 p1 = make_float2(v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y);
        const float2 p2 = make_float2(v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y);
        // q1 = s*i*(s1 b1 + s2 b2), q2 = s*i*(s2 b1 - s1 b2)
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
    __device__ static void run(float2 (&v)[8], const float2* tw, int n, float s) {
        float2 e[4] = {v[0], v[2], v[4], v[6]};
        float2 o[4] = {v[1], v[3], v[5], v[7]};
        Dft<4>::run(e, tw, n, s);
        Dft<4>::run(o, tw, n, s);
        const float r = 0.70710678118654752440f;
        // W8^k for forward (s=-1): (r,-r), -i, (-r,-r); inverse conjugates
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

// One out-of-place Stockham pass of radix R over `nrings` rings of length n
// (src -> dst, both in SMEM): each thread loads R points, applies the twiddles,
// runs the radix-R DFT in registers and stores R points.
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
                float2 w = tw[k * r * tstride];
                if (s > 0) w.y = -w.y;
                x = cmul(x, w);
            }
            v[r] = x;
        }
        Dft<R>::run(v, tw, n, s);
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

// Runs all passes ping-ponging between a and b; returns the buffer holding the result.
__device__ __forceinline__ float2* fft_rings(float2* a, float2* b, int nrings, const FftArgs& fa,
                                             const float2* tw, float s) {
    int ns = 1;
    for (int st = 0; st < fa.nstages; ++st) {
        const int R = fa.radix[st];
        switch (R) {
            case 2: stockham_pass<2>(a, b, nrings, fa.n, ns, tw, s); break;
            case 3: stockham_pass<3>(a, b, nrings, fa.n, ns, tw, s); break;
            case 4: stockham_pass<4>(a, b, nrings, fa.n, ns, tw, s); break;
            case 5: stockham_pass<5>(a, b, nrings, fa.n, ns, tw, s); break;
            case 8: stockham_pass<8>(a, b, nrings, fa.n, ns, tw, s); break;
            default: break;
        }
        ns *= R;
        float2* t = a;
        a = b;
        b = t;
    }
    return a;
}

__device__ __forceinline__ void load_twiddles(float2* tw_s, const float2* __restrict__ tw, int n) {
    for (int i = threadIdx.x; i < n; i += FFT_THREADS) tw_s[i] = tw[i];
}

// ---------------------------------------------------------------- forward fold
__global__ void __launch_bounds__(FFT_THREADS) fft_fwd_fold_kernel(
    FftArgs a, const float2* __restrict__ tw, const float* __restrict__ x,
    const int2* __restrict__ rows, int R, int rpb, int nlat, int mmax, float* __restrict__ eo,
    int64_t ld_eo, int64_t twoF) {
    extern __shared__ float2 sm[];
    const int n = a.n;
    float2* tw_s = sm;
    float2* buf = sm + n;
    float2* buf2 = buf + rpb * n;
    const int r0 = blockIdx.x * rpb;
    const int f = blockIdx.y;
    const int nr = min(rpb, R - r0);
    load_twiddles(tw_s, tw, n);
    const float* xf = x + static_cast<int64_t>(f) * nlat * n;
    for (int j = 0; j < nr; ++j) {
        const int2 rw = rows[r0 + j];
        const float* pa = xf + static_cast<int64_t>(rw.x) * n;
        const float* pb = rw.y >= 0 ? xf + static_cast<int64_t>(rw.y) * n : nullptr;
        if ((n & 3) == 0) {
            for (int k4 = threadIdx.x; k4 < n / 4; k4 += FFT_THREADS) {
                const float4 va = __ldg(reinterpret_cast<const float4*>(pa) + k4);
                const float4 vb = pb ? __ldg(reinterpret_cast<const float4*>(pb) + k4)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                float2* d = buf + j * n + 4 * k4;
                d[0] = make_float2(va.x, vb.x);
                d[1] = make_float2(va.y, vb.y);
                d[2] = make_float2(va.z, vb.z);
                d[3] = make_float2(va.w, vb.w);
            }
        } else {
            for (int k = threadIdx.x; k < n; k += FFT_THREADS)
                buf[j * n + k] = make_float2(pa[k], pb ? pb[k] : 0.f);
        }
    }
    __syncthreads();
    buf = fft_rings(buf, buf2, nr, a, tw_s, -1.f);
    // epilogue: E/O bins m < mmax -> eo[(m*2+p)*2F + 2f + reim][r0 + j]
    const int total = mmax * 4 * rpb;
    for (int o = threadIdx.x; o < total; o += FFT_THREADS) {
        const int j = o % rpb;
        const int q = (o / rpb) & 3;
        const int m = o / (4 * rpb);
        if (j >= nr) continue;
        const float2 z = buf[j * n + m];
        const float2 zc = buf[j * n + (m == 0 ? 0 : n - m)];
        // A = (Z + conj Zc)/2, B = (Z - conj Zc)/(2i); E = A + B, O = A - B
        const float ar = 0.5f * (z.x + zc.x), ai = 0.5f * (z.y - zc.y);
        const float br = 0.5f * (z.y + zc.y), bi = -0.5f * (z.x - zc.x);
        const int p = q >> 1, reim = q & 1;
        const float val = p == 0 ? (reim ? ai + bi : ar + br) : (reim ? ai - bi : ar - br);
        eo[((static_cast<int64_t>(m) * 2 + p) * twoF + 2 * f + reim) * ld_eo + r0 + j] = val;
    }
}

// -------------------------------------------------------------- inverse unfold
__global__ void __launch_bounds__(FFT_THREADS) fft_inv_unfold_kernel(
    FftArgs a, const float2* __restrict__ tw, const float* __restrict__ eoi,
    const int2* __restrict__ rows, int R, int rpb, int nlat, int msynth, int lmax,
    int64_t ld_eo, int64_t twoF, float* __restrict__ y) {
    extern __shared__ float2 sm[];
    const int n = a.n;
    float2* tw_s = sm;
    float2* buf = sm + n;
    float2* buf2 = buf + rpb * n;
    const int r0 = blockIdx.x * rpb;
    const int f = blockIdx.y;
    const int nr = min(rpb, R - r0);
    load_twiddles(tw_s, tw, n);
    for (int i = threadIdx.x; i < nr * n; i += FFT_THREADS) buf[i] = make_float2(0.f, 0.f);
    __syncthreads();
    for (int o = threadIdx.x; o < msynth * rpb; o += FFT_THREADS) {
        const int j = o % rpb;
        const int m = o / rpb;
        if (j >= nr) continue;
        const int2 rw = rows[r0 + j];
        const int64_t c = r0 + j;
        const int64_t g0 = (static_cast<int64_t>(m) * 2 + 0) * twoF + 2 * f;
        const int64_t g1 = (static_cast<int64_t>(m) * 2 + 1) * twoF + 2 * f;
        const int l0 = (lmax - m + 1) / 2, l1 = (lmax - m) / 2;  // L_{m,0}, L_{m,1}
        float2 ev = make_float2(0.f, 0.f), od = make_float2(0.f, 0.f);
        if (l0 > 0) ev = make_float2(eoi[g0 * ld_eo + c], eoi[(g0 + 1) * ld_eo + c]);
        if (l1 > 0) od = make_float2(eoi[g1 * ld_eo + c], eoi[(g1 + 1) * ld_eo + c]);
        const float2 ha = cadd(ev, od);
        const float2 hb = rw.y >= 0 ? csub(ev, od) : make_float2(0.f, 0.f);
        if (m == 0) {
            buf[j * n] = make_float2(ha.x, hb.x);  // Im of the DC bin is dropped
        } else {
            buf[j * n + m] = make_float2(ha.x - hb.y, ha.y + hb.x);      // ha + i hb
            buf[j * n + n - m] = make_float2(ha.x + hb.y, hb.x - ha.y);  // conj ha + i conj hb
        }
    }
    __syncthreads();
    buf = fft_rings(buf, buf2, nr, a, tw_s, 1.f);
    float* yf = y + static_cast<int64_t>(f) * nlat * n;
    for (int j = 0; j < nr; ++j) {
        const int2 rw = rows[r0 + j];
        float* pa = yf + static_cast<int64_t>(rw.x) * n;
        float* pb = rw.y >= 0 ? yf + static_cast<int64_t>(rw.y) * n : nullptr;
        if ((n & 3) == 0) {
            for (int k4 = threadIdx.x; k4 < n / 4; k4 += FFT_THREADS) {
                const float2* s = buf + j * n + 4 * k4;
                reinterpret_cast<float4*>(pa)[k4] = make_float4(s[0].x, s[1].x, s[2].x, s[3].x);
                if (pb)
                    reinterpret_cast<float4*>(pb)[k4] = make_float4(s[0].y, s[1].y, s[2].y, s[3].y);
            }
        } else {
            for (int k = threadIdx.x; k < n; k += FFT_THREADS) {
                pa[k] = buf[j * n + k].x;
                if (pb) pb[k] = buf[j * n + k].y;
            }
        }
    }
}

// ----------------------------------------------------------------- plain (dist)
__global__ void __launch_bounds__(FFT_THREADS) fft_fwd_plain_kernel(
    FftArgs a, const float2* __restrict__ tw, const float* __restrict__ rings, int64_t nrings,
    int rpb, int nbins, float scale, float2* __restrict__ bins) {
    extern __shared__ float2 sm[];
    const int n = a.n;
    float2* tw_s = sm;
    float2* buf = sm + n;
    float2* buf2 = buf + rpb * n;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * rpb;  // complex row = 2 real rings
    const int64_t ncomplex = (nrings + 1) / 2;
    const int nr = static_cast<int>(min(static_cast<int64_t>(rpb), ncomplex - c0));
    load_twiddles(tw_s, tw, n);
    for (int i = threadIdx.x; i < nr * n; i += FFT_THREADS) {
        const int j = i / n, k = i - j * n;
        const int64_t ra = 2 * (c0 + j), rb = ra + 1;
        buf[i] = make_float2(rings[ra * n + k], rb < nrings ? rings[rb * n + k] : 0.f);
    }
    __syncthreads();
    buf = fft_rings(buf, buf2, nr, a, tw_s, -1.f);
    for (int o = threadIdx.x; o < nr * 2 * nbins; o += FFT_THREADS) {
        const int m = o % nbins;
        const int jj = o / nbins;  // real ring within the block
        const int j = jj >> 1, which = jj & 1;
        const int64_t ring = 2 * (c0 + j) + which;
        if (ring >= nrings) continue;
        const float2 z = buf[j * n + m];
        const float2 zc = buf[j * n + (m == 0 ? 0 : n - m)];
        float2 v;
        if (which == 0)
            v = make_float2(0.5f * (z.x + zc.x), 0.5f * (z.y - zc.y));
        else
            v = make_float2(0.5f * (z.y + zc.y), -0.5f * (z.x - zc.x));
        bins[ring * nbins + m] = make_float2(v.x * scale, v.y * scale);
    }
}

// O(n^2) fallback for lengths with a prime factor > 13 (correct, slow).
__global__ void dft_direct_kernel(const float2* __restrict__ tw, int n, float2* __restrict__ buf_in,
                                  float2* __restrict__ buf_out, int64_t nrings, float s) {
    const int64_t ring = blockIdx.y;
    if (ring >= nrings) return;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        float2 acc = make_float2(0.f, 0.f);
        for (int j = 0; j < n; ++j) {
            float2 w = tw[static_cast<int64_t>(j) * k % n];
            if (s > 0) w.y = -w.y;
            acc = cadd(acc, cmul(buf_in[ring * n + j], w));
        }
        buf_out[ring * n + k] = acc;
    }
}


// ------------------------------------------------------------- plain inverse
__global__ void __launch_bounds__(FFT_THREADS) fft_inv_plain_kernel(
    FftArgs a, const float2* __restrict__ tw, const float2* __restrict__ bins, int64_t nrings,
    int rpb, int nbins, float scale, float* __restrict__ rings) {
    extern __shared__ float2 sm[];
    const int n = a.n;
    float2* tw_s = sm;
    float2* buf = sm + n;
    float2* buf2 = buf + rpb * n;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * rpb;
    const int64_t ncomplex = (nrings + 1) / 2;
    const int nr = static_cast<int>(min(static_cast<int64_t>(rpb), ncomplex - c0));
    load_twiddles(tw_s, tw, n);
    const int half = n / 2;
    for (int i = threadIdx.x; i < nr * n; i += FFT_THREADS) {
        const int j = i / n, k = i - j * n;
        const int64_t ra = 2 * (c0 + j), rb = ra + 1;
        const int kk = k <= half ? k : n - k;
        float2 ha = make_float2(0.f, 0.f), hb = make_float2(0.f, 0.f);
        if (kk < nbins) {
            ha = bins[ra * nbins + kk];
            if (rb < nrings) hb = bins[rb * nbins + kk];
        }
        if (kk == 0 || 2 * kk == n) { ha.y = 0.f; hb.y = 0.f; }
        if (k > half) { ha.y = -ha.y; hb.y = -hb.y; }
        buf[i] = make_float2(ha.x - hb.y, ha.y + hb.x);
    }
    __syncthreads();
    buf = fft_rings(buf, buf2, nr, a, tw_s, 1.f);
    for (int i = threadIdx.x; i < nr * 2 * n; i += FFT_THREADS) {
        const int jj = i / n, k = i - jj * n;
        const int j = jj >> 1, which = jj & 1;
        const int64_t ring = 2 * (c0 + j) + which;
        if (ring >= nrings) continue;
        const float2 z = buf[j * n + k];
        rings[ring * n + k] = (which ? z.y : z.x) * scale;
    }
}

// ---------------------------------------------- channel-minor forward (DISCO)
// block: (c-tile of 2*rpb channels, input row hi, batch b)
__global__ void __launch_bounds__(FFT_THREADS) fft_fwd_cminor_kernel(
    FftArgs a, const float2* __restrict__ tw, const float* __restrict__ x, int64_t C, int64_t H,
    int rpb, int nbins, float2* __restrict__ U) {
    extern __shared__ float2 sm[];
    const int n = a.n;
    float2* tw_s = sm;
    float2* buf = sm + n;
    float2* buf2 = buf + rpb * n;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 2 * rpb;
    const int64_t hi = blockIdx.y, b = blockIdx.z;
    const int nch = static_cast<int>(min(static_cast<int64_t>(2 * rpb), C - c0));
    const int nr = (nch + 1) / 2;
    load_twiddles(tw_s, tw, n);
    for (int i = threadIdx.x; i < nr * n; i += FFT_THREADS) {
        const int j = i / n, k = i - j * n;
        const int64_t ca = c0 + 2 * j, cb = ca + 1;
        const float va = x[((b * C + ca) * H + hi) * n + k];
        const float vb = cb < c0 + nch ? x[((b * C + cb) * H + hi) * n + k] : 0.f;
        buf[i] = make_float2(va, vb);
    }
    __syncthreads();
    buf = fft_rings(buf, buf2, nr, a, tw_s, -1.f);
    float2* Ub = U + (b * H + hi) * static_cast<int64_t>(nbins) * C;
    for (int o = threadIdx.x; o < nbins * 2 * rpb; o += FFT_THREADS) {
        const int cl = o % (2 * rpb);
        const int m = o / (2 * rpb);
        if (cl >= nch) continue;
        const int j = cl >> 1;
        const float2 z = buf[j * n + m];
        const float2 zc = buf[j * n + (m == 0 ? 0 : n - m)];
        const float2 v = (cl & 1) ? make_float2(0.5f * (z.y + zc.y), -0.5f * (z.x - zc.x))
                                  : make_float2(0.5f * (z.x + zc.x), 0.5f * (z.y - zc.y));
        Ub[static_cast<int64_t>(m) * C + c0 + cl] = v;
    }
}

__global__ void dft_rows_generic_kernel(const float2* __restrict__ tw, int n, const float* __restrict__ rings,
                                        int64_t nrings, int nbins, float2* __restrict__ out) {
    // out[ring][m] = sum_j rings[ring][j] W^{jm}   (direct, for odd radices)
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrings * nbins) return;
    const int m = static_cast<int>(i % nbins);
    const int64_t ring = i / nbins;
    float2 acc = make_float2(0.f, 0.f);
    for (int j = 0; j < n; ++j) {
        const float2 w = tw[static_cast<int64_t>(j) * m % n];
        const float v = rings[ring * n + j];
        acc.x += v * w.x;
        acc.y += v * w.y;
    }
    out[i] = acc;
}

__global__ void idft_rows_generic_kernel(const float2* __restrict__ tw, int n, const float2* __restrict__ bins,
                                         int64_t nrings, int nbins, float scale, float* __restrict__ rings) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrings * n) return;
    const int k = static_cast<int>(i % n);
    const int64_t ring = i / n;
    const int half = n / 2;
    float acc = 0.f;
    for (int m = 0; m < nbins && m <= half; ++m) {
        float2 h = bins[ring * nbins + m];
        if (m == 0 || 2 * m == n) h.y = 0.f;
        const float2 w = tw[static_cast<int64_t>(k) * m % n];  // e^{-i..}; inverse uses conj
        const float re = h.x * w.x + h.y * w.y;             // Re(h * conj(w))
        acc += (m == 0 || 2 * m == n) ? re : 2.f * re;
    }
    rings[i] = acc * scale;
}

__global__ void transpose_cminor_kernel(const float2* __restrict__ in, int64_t B, int64_t C,
                                        int64_t H, int nbins, float2* __restrict__ U) {
    // in [B][C][H][nbins] -> U [B][H][nbins][C]
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t per_b = C * H * nbins;
    if (i >= B * per_b) return;
    const int64_t b = i / per_b;
    const int64_t r = i % per_b;
    const int64_t c = r % C;
    const int64_t m = (r / C) % nbins;
    const int64_t h = r / (C * nbins);
    U[i] = in[((b * C + c) * H + h) * nbins + m];
}

FftArgs make_args(const FftPlan& fp) {
    FftArgs a;
    a.n = fp.n;
    a.nstages = fp.nstages;
    for (int i = 0; i < FFT_MAX_STAGES; ++i) a.radix[i] = fp.radix[i];
    return a;
}

size_t smem_bytes(const FftPlan& fp) {
    return static_cast<size_t>(fp.n) * sizeof(float2) * (1 + 2 * fp.rows_per_block);
}

void set_smem(const void* fn, size_t bytes) {
    SPH_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
}

}  // namespace

void FftPlan::build(int n_) {
    n = n_;
    require(n >= 1, "fft: length must be >= 1");
    nstages = 0;
    direct = false;
    int m = n;
    // prefer radix 8 and 4, then 2, 3, 5; other primes use the O(n^2) fallback
    while (m % 8 == 0 && m != 1) { radix[nstages++] = 8; m /= 8; }
    while (m % 4 == 0) { radix[nstages++] = 4; m /= 4; }
    while (m % 2 == 0) { radix[nstages++] = 2; m /= 2; }
    for (int p : {3, 5})
        while (m % p == 0) { radix[nstages++] = p; m /= p; }
    if (m != 1 || nstages > FFT_MAX_STAGES) direct = true;
    std::vector<float2> h(n);
    for (int q = 0; q < n; ++q) {
        const double ang = -2.0 * M_PI * static_cast<double>(q) / static_cast<double>(n);
        h[q] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
    }
    tw.alloc(n, false);
    SPH_CUDA(cudaMemcpy(tw.p, h.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
    // complex rings per CTA: ping-pong buffers + twiddles within ~110 KB so two CTAs
    // share an SM; at most 16
    int rpb = 16;
    while (rpb > 1 && static_cast<size_t>(n) * sizeof(float2) * (1 + 2 * rpb) > 110 * 1024) --rpb;
    rows_per_block = rpb;
    if (static_cast<size_t>(n) * sizeof(float2) * (1 + 2 * rows_per_block) > 200 * 1024) direct = true;
    if (direct) rows_per_block = 1;
}

// Direct-DFT fallback: run the O(n^2) transform on a global scratch ring buffer.
// Only used for ring lengths whose factorisation has primes > 13 (never at the
// benchmark sizes).  Implemented by staging through a temporary buffer.
static void direct_transform(const FftPlan& fp, float2* data, int64_t nrings, float s,
                             cudaStream_t st) {
    DevBuf<float2> tmp(static_cast<size_t>(nrings) * fp.n, false);
    dim3 grid((fp.n + 127) / 128, static_cast<unsigned>(nrings));
    dft_direct_kernel<<<grid, 128, 0, st>>>(fp.tw.p, fp.n, data, tmp.p, nrings, s);
    SPH_LAUNCH_CHECK();
    count_launch();
    SPH_CUDA(cudaMemcpyAsync(data, tmp.p, tmp.bytes(), cudaMemcpyDeviceToDevice, st));
    SPH_CUDA(cudaStreamSynchronize(st));
}

__global__ void pack_pairs_kernel(const float* __restrict__ x, const int2* __restrict__ rows,
                                  int R, int nlat, int n, int64_t F, float2* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = F * R * static_cast<int64_t>(n);
    if (i >= total) return;
    const int k = static_cast<int>(i % n);
    const int r = static_cast<int>((i / n) % R);
    const int64_t f = i / (static_cast<int64_t>(n) * R);
    const int2 rw = rows[r];
    const float* xf = x + f * nlat * n;
    out[i] = make_float2(xf[static_cast<int64_t>(rw.x) * n + k],
                         rw.y >= 0 ? xf[static_cast<int64_t>(rw.y) * n + k] : 0.f);
}

__global__ void fold_out_kernel(const float2* __restrict__ z, int R, int n, int64_t F, int mmax,
                                float* __restrict__ eo, int64_t ld_eo) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = F * R * static_cast<int64_t>(mmax);
    if (i >= total) return;
    const int r = static_cast<int>(i % R);
    const int m = static_cast<int>((i / R) % mmax);
    const int64_t f = i / (static_cast<int64_t>(R) * mmax);
    const float2* zr = z + (f * R + r) * n;
    const float2 a = zr[m], b = zr[m == 0 ? 0 : n - m];
    const float ar = 0.5f * (a.x + b.x), ai = 0.5f * (a.y - b.y);
    const float br = 0.5f * (a.y + b.y), bi = -0.5f * (a.x - b.x);
    const int64_t twoF = 2 * F;
    eo[((static_cast<int64_t>(m) * 2 + 0) * twoF + 2 * f) * ld_eo + r] = ar + br;
    eo[((static_cast<int64_t>(m) * 2 + 0) * twoF + 2 * f + 1) * ld_eo + r] = ai + bi;
    eo[((static_cast<int64_t>(m) * 2 + 1) * twoF + 2 * f) * ld_eo + r] = ar - br;
    eo[((static_cast<int64_t>(m) * 2 + 1) * twoF + 2 * f + 1) * ld_eo + r] = ai - bi;
}

void fft_forward_fold(const FftPlan& fp, const FoldRows& fr, const float* x, int64_t F, int nlat,
                      int mmax, float* eo, int64_t ld_eo, cudaStream_t st) {
    if (F == 0) return;
    if (fp.direct) {
        DevBuf<float2> z(static_cast<size_t>(F) * fr.R * fp.n, false);
        const int64_t tot = F * fr.R * static_cast<int64_t>(fp.n);
        pack_pairs_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(
            x, fr.d_rows.p, fr.R, nlat, fp.n, F, z.p);
        SPH_LAUNCH_CHECK();
        count_launch();
        direct_transform(fp, z.p, F * fr.R, -1.f, st);
        const int64_t tot2 = F * fr.R * static_cast<int64_t>(mmax);
        fold_out_kernel<<<static_cast<unsigned>((tot2 + 255) / 256), 256, 0, st>>>(
            z.p, fr.R, fp.n, F, mmax, eo, ld_eo);
        SPH_LAUNCH_CHECK();
        count_launch();
        SPH_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const size_t sm = smem_bytes(fp);
    static bool once = (set_smem(reinterpret_cast<const void*>(fft_fwd_fold_kernel), 200 * 1024), true);
    (void)once;
    require(F <= 65535, "fft: at most 65535 fields per call");
    dim3 grid((fr.R + fp.rows_per_block - 1) / fp.rows_per_block, static_cast<unsigned>(F));
    ProfScope prof("fft_fwd_fold", st, 4.0 * F * (static_cast<double>(nlat) * fp.n + 4.0 * mmax * fr.R));
    fft_fwd_fold_kernel<<<grid, FFT_THREADS, sm, st>>>(make_args(fp), fp.tw.p, x, fr.d_rows.p,
                                                        fr.R, fp.rows_per_block, nlat, mmax, eo,
                                                        ld_eo, 2 * F);
    SPH_LAUNCH_CHECK();
    count_launch();
}

__global__ void unfold_in_kernel(const float* __restrict__ eoi, const int2* __restrict__ rows,
                                 int R, int n, int64_t F, int msynth, int lmax, int64_t ld_eo,
                                 float2* __restrict__ z) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = F * R * static_cast<int64_t>(n);
    if (i >= total) return;
    const int k = static_cast<int>(i % n);
    const int r = static_cast<int>((i / n) % R);
    const int64_t f = i / (static_cast<int64_t>(n) * R);
    const int m = k < msynth ? k : (n - k < msynth ? n - k : -1);
    float2 out = make_float2(0.f, 0.f);
    if (m >= 0) {
        const int64_t twoF = 2 * F;
        const int64_t g0 = (static_cast<int64_t>(m) * 2) * twoF + 2 * f;
        const int64_t g1 = (static_cast<int64_t>(m) * 2 + 1) * twoF + 2 * f;
        const int l0 = (lmax - m + 1) / 2, l1 = (lmax - m) / 2;
        float2 ev = make_float2(0.f, 0.f), od = make_float2(0.f, 0.f);
        if (l0 > 0) ev = make_float2(eoi[g0 * ld_eo + r], eoi[(g0 + 1) * ld_eo + r]);
        if (l1 > 0) od = make_float2(eoi[g1 * ld_eo + r], eoi[(g1 + 1) * ld_eo + r]);
        const float2 ha = cadd(ev, od);
        const float2 hb = rows[r].y >= 0 ? csub(ev, od) : make_float2(0.f, 0.f);
        if (m == 0)
            out = make_float2(ha.x, hb.x);
        else if (k == m)
            out = make_float2(ha.x - hb.y, ha.y + hb.x);
        else
            out = make_float2(ha.x + hb.y, hb.x - ha.y);
    }
    z[i] = out;
}

__global__ void unpack_pairs_kernel(const float2* __restrict__ z, const int2* __restrict__ rows,
                                    int R, int nlat, int n, int64_t F, float* __restrict__ y) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = F * R * static_cast<int64_t>(n);
    if (i >= total) return;
    const int k = static_cast<int>(i % n);
    const int r = static_cast<int>((i / n) % R);
    const int64_t f = i / (static_cast<int64_t>(n) * R);
    const int2 rw = rows[r];
    float* yf = y + f * nlat * n;
    yf[static_cast<int64_t>(rw.x) * n + k] = z[i].x;
    if (rw.y >= 0) yf[static_cast<int64_t>(rw.y) * n + k] = z[i].y;
}

void fft_inverse_unfold(const FftPlan& fp, const FoldRows& fr, const float* eoi, int64_t F,
                        int nlat, int mmax, int msynth, int lmax, int64_t ld_eo, float* y,
                        cudaStream_t st) {
    (void)mmax;
    if (F == 0) return;
    if (fp.direct) {
        DevBuf<float2> z(static_cast<size_t>(F) * fr.R * fp.n, false);
        const int64_t tot = F * fr.R * static_cast<int64_t>(fp.n);
        unfold_in_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(
            eoi, fr.d_rows.p, fr.R, fp.n, F, msynth, lmax, ld_eo, z.p);
        SPH_LAUNCH_CHECK();
        count_launch();
        direct_transform(fp, z.p, F * fr.R, 1.f, st);
        unpack_pairs_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(
            z.p, fr.d_rows.p, fr.R, nlat, fp.n, F, y);
        SPH_LAUNCH_CHECK();
        count_launch();
        SPH_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const size_t sm = smem_bytes(fp);
    static bool once = (set_smem(reinterpret_cast<const void*>(fft_inv_unfold_kernel), 200 * 1024), true);
    (void)once;
    require(F <= 65535, "fft: at most 65535 fields per call");
    dim3 grid((fr.R + fp.rows_per_block - 1) / fp.rows_per_block, static_cast<unsigned>(F));
    ProfScope prof("fft_inv_unfold", st, 4.0 * F * (static_cast<double>(nlat) * fp.n + 4.0 * msynth * fr.R));
    fft_inv_unfold_kernel<<<grid, FFT_THREADS, sm, st>>>(make_args(fp), fp.tw.p, eoi, fr.d_rows.p,
                                                          fr.R, fp.rows_per_block, nlat, msynth,
                                                          lmax, ld_eo, 2 * F, y);
    SPH_LAUNCH_CHECK();
    count_launch();
}

__global__ void plain_pack_kernel(const float* __restrict__ rings, int64_t nrings, int n,
                                  float2* __restrict__ z) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nc = (nrings + 1) / 2;
    if (i >= nc * n) return;
    const int64_t j = i / n;
    const int k = static_cast<int>(i % n);
    const int64_t ra = 2 * j, rb = ra + 1;
    z[i] = make_float2(rings[ra * n + k], rb < nrings ? rings[rb * n + k] : 0.f);
}

__global__ void plain_out_kernel(const float2* __restrict__ z, int64_t nrings, int n, int nbins,
                                 float scale, float2* __restrict__ bins) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrings * nbins) return;
    const int m = static_cast<int>(i % nbins);
    const int64_t ring = i / nbins;
    const float2* zr = z + (ring / 2) * n;
    const float2 a = zr[m], b = zr[m == 0 ? 0 : n - m];
    float2 v = (ring & 1) ? make_float2(0.5f * (a.y + b.y), -0.5f * (a.x - b.x))
                          : make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
    bins[i] = make_float2(v.x * scale, v.y * scale);
}

void fft_forward_plain(const FftPlan& fp, const float* rings, int64_t nrings, int nbins,
                       float scale, float2* bins, cudaStream_t st) {
    if (nrings == 0) return;
    if (fp.direct) {
        const int64_t nc = (nrings + 1) / 2;
        DevBuf<float2> z(static_cast<size_t>(nc) * fp.n, false);
        plain_pack_kernel<<<static_cast<unsigned>((nc * fp.n + 255) / 256), 256, 0, st>>>(
            rings, nrings, fp.n, z.p);
        SPH_LAUNCH_CHECK();
        count_launch();
        direct_transform(fp, z.p, nc, -1.f, st);
        plain_out_kernel<<<static_cast<unsigned>((nrings * nbins + 255) / 256), 256, 0, st>>>(
            z.p, nrings, fp.n, nbins, scale, bins);
        SPH_LAUNCH_CHECK();
        count_launch();
        SPH_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const size_t sm = smem_bytes(fp);
    static bool once = (set_smem(reinterpret_cast<const void*>(fft_fwd_plain_kernel), 200 * 1024), true);
    (void)once;
    const int64_t nc = (nrings + 1) / 2;
    const int64_t nblk = (nc + fp.rows_per_block - 1) / fp.rows_per_block;
    require(nblk < (1LL << 31), "fft: too many rings");
    ProfScope prof("fft_fwd_plain", st, 4.0 * nrings * (fp.n + 2.0 * nbins));
    fft_fwd_plain_kernel<<<static_cast<unsigned>(nblk), FFT_THREADS, sm, st>>>(
        make_args(fp), fp.tw.p, rings, nrings, fp.rows_per_block, nbins, scale, bins);
    SPH_LAUNCH_CHECK();
    count_launch();
}

void fft_inverse_plain(const FftPlan& fp, const float2* bins, int64_t nrings, int nbins,
                       float scale, float* rings, cudaStream_t st) {
    if (nrings == 0) return;
    if (fp.direct) {
        const int64_t tot = nrings * fp.n;
        idft_rows_generic_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(
            fp.tw.p, fp.n, bins, nrings, nbins, scale, rings);
        SPH_LAUNCH_CHECK();
        count_launch();
        return;
    }
    const size_t sm = smem_bytes(fp);
    static bool once = (set_smem(reinterpret_cast<const void*>(fft_inv_plain_kernel), 200 * 1024), true);
    (void)once;
    const int64_t nc = (nrings + 1) / 2;
    const int64_t nblk = (nc + fp.rows_per_block - 1) / fp.rows_per_block;
    ProfScope prof("fft_inv_plain", st, 4.0 * nrings * (fp.n + 2.0 * nbins));
    fft_inv_plain_kernel<<<static_cast<unsigned>(nblk), FFT_THREADS, sm, st>>>(
        make_args(fp), fp.tw.p, bins, nrings, fp.rows_per_block, nbins, scale, rings);
    SPH_LAUNCH_CHECK();
    count_launch();
}

void fft_forward_cminor(const FftPlan& fp, const float* x, int64_t B, int64_t C, int64_t H,
                        int nbins, float2* U, cudaStream_t st) {
    if (B * C * H == 0) return;
    if (fp.direct) {
        DevBuf<float2> tmp(static_cast<size_t>(B * C * H) * nbins, false);
        const int64_t tot = B * C * H * nbins;
        dft_rows_generic_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(
            fp.tw.p, fp.n, x, B * C * H, nbins, tmp.p);
        SPH_LAUNCH_CHECK();
        transpose_cminor_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(
            tmp.p, B, C, H, nbins, U);
        SPH_LAUNCH_CHECK();
        count_launch(2);
        SPH_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const size_t sm = smem_bytes(fp);
    static bool once = (set_smem(reinterpret_cast<const void*>(fft_fwd_cminor_kernel), 200 * 1024), true);
    (void)once;
    require(H <= 65535 && B <= 65535, "disco fft: too many rows");
    dim3 grid(static_cast<unsigned>((C + 2 * fp.rows_per_block - 1) / (2 * fp.rows_per_block)),
              static_cast<unsigned>(H), static_cast<unsigned>(B));
    ProfScope prof("fft_fwd_cminor", st, 4.0 * B * C * H * (fp.n + 2.0 * nbins));
    fft_fwd_cminor_kernel<<<grid, FFT_THREADS, sm, st>>>(make_args(fp), fp.tw.p, x, C, H,
                                                          fp.rows_per_block, nbins, U);
    SPH_LAUNCH_CHECK();
    count_launch();
}

}  // namespace sph
