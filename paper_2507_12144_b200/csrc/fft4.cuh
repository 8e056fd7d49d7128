// Register-resident four-step FFT for the benchmark ring lengths (N = N1 * N2 with
// N2 = 45: 1440 = 32*45, 720 = 16*45, 360 = 8*45, 180 = 4*45).
//
//   n = n2 + N2*n1,  k = k1 + N1*k2
//   phase A (item = ring, n2):  Y[n2][k1] = W_N^{n2 k1} * sum_n1 x[n2 + N2 n1] W_N1^{n1 k1}
//   phase B (item = ring, k1):  X[k1 + N1 k2] = sum_n2 Y[n2][k1] W_N2^{n2 k2}
// Sub-DFTs run fully unrolled in registers with compile-time twiddles (constexpr trig);
// phase A works in place (an item reads and writes the same N1 slots), phase B stages
// its N2 values in registers across one barrier.  Two shared-memory exchanges per
// transform instead of one per radix pass.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace sph {
namespace fft4 {

constexpr int THREADS = 256;

// ---------------------------------------------------------- compile-time trig
constexpr double kPi = 3.14159265358979323846264338327950288;
__host__ __device__ constexpr double sin_red(double x) {  // |x| <= pi/4
    double x2 = x * x, term = x, sum = x;
    for (int i = 1; i < 14; ++i) {
        term *= -x2 / ((2.0 * i) * (2.0 * i + 1.0));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double cos_red(double x) {
    double x2 = x * x, term = 1.0, sum = 1.0;
    for (int i = 1; i < 14; ++i) {
        term *= -x2 / ((2.0 * i - 1.0) * (2.0 * i));
        sum += term;
    }
    return sum;
}
struct cxf {
    float x, y;
};
// exp(-2 pi i q / n), octant-reduced so the series stays within |x| <= pi/4
__host__ __device__ constexpr cxf twiddle(int q, int n) {
    q %= n;
    if (q < 0) q += n;
    const long long e = 8LL * q;
    const int oct = static_cast<int>(e / n);
    const double r = (static_cast<double>(e - static_cast<long long>(oct) * n) / n) * (kPi / 4);
    const double cr = cos_red(r), sr = sin_red(r);
    const double cq = cos_red(kPi / 4 - r), sq = sin_red(kPi / 4 - r);
    double c = 0, s = 0;
    switch (oct) {
        case 0: c = cr; s = sr; break;
        case 1: c = sq; s = cq; break;
        case 2: c = -sr; s = cr; break;
        case 3: c = -cq; s = sq; break;
        case 4: c = -cr; s = -sr; break;
        case 5: c = -sq; s = -cq; break;
        case 6: c = sr; s = -cr; break;
        default: c = cq; s = -sq; break;
    }
    return cxf{static_cast<float>(c), static_cast<float>(-s)};
}

template <int I0, int I1, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (I0 < I1) {
        f(std::integral_constant<int, I0>{});
        static_for<I0 + 1, I1>(f);
    }
}

__device__ __forceinline__ float2 add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// a * exp(-+2 pi i Q / N): exact quadrant rotations, constant twiddle otherwise
template <int Q, int N, bool INV>
__device__ __forceinline__ float2 rot(float2 a) {
    constexpr int q = ((Q % N) + N) % N;
    if constexpr (q == 0) {
        return a;
    } else if constexpr ((4 * q) % N == 0) {
        constexpr int quad = 4 * q / N;
        if constexpr (quad == 2) return make_float2(-a.x, -a.y);
        else if constexpr ((quad == 1) != INV) return make_float2(a.y, -a.x);  // * (-i)
        else return make_float2(-a.y, a.x);                                   // * (+i)
    } else {
        constexpr cxf w = twiddle(q, N);
        constexpr float wy = INV ? -w.y : w.y;
        return make_float2(a.x * w.x - a.y * wy, a.x * wy + a.y * w.x);
    }
}

__host__ __device__ constexpr int first_factor(int n) {
    return n % 4 == 0 ? 4 : n % 2 == 0 ? 2 : n % 3 == 0 ? 3 : n % 5 == 0 ? 5 : n;
}

// In-register DFT of size N over v[OFF + S*i], i < N.
template <int M, int N, int OFF, int S, bool INV>
__device__ __forceinline__ void dft(float2 (&v)[M]) {
    if constexpr (N == 1) {
        return;
    } else if constexpr (N == 2) {
        const float2 a = v[OFF], b = v[OFF + S];
        v[OFF] = add(a, b);
        v[OFF + S] = sub(a, b);
    } else if constexpr (N == 4) {
        const float2 t0 = add(v[OFF], v[OFF + 2 * S]), t1 = sub(v[OFF], v[OFF + 2 * S]);
        const float2 t2 = add(v[OFF + S], v[OFF + 3 * S]);
        const float2 t3 = rot<1, 4, INV>(sub(v[OFF + S], v[OFF + 3 * S]));
        v[OFF] = add(t0, t2);
        v[OFF + 2 * S] = sub(t0, t2);
        v[OFF + S] = add(t1, t3);
        v[OFF + 3 * S] = sub(t1, t3);
    } else if constexpr (N == 3) {
        const float2 x0 = v[OFF], x1 = v[OFF + S], x2 = v[OFF + 2 * S];
        const float2 t = add(x1, x2), d = sub(x1, x2);
        const float2 m = make_float2(x0.x - 0.5f * t.x, x0.y - 0.5f * t.y);
        const float k = 0.86602540378443864676f;
        // forward: X1 = m - i k d, X2 = m + i k d
        const float2 ikd = INV ? make_float2(-k * d.y, k * d.x) : make_float2(k * d.y, -k * d.x);
        v[OFF] = add(x0, t);
        v[OFF + S] = add(m, ikd);
        v[OFF + 2 * S] = sub(m, ikd);
    } else if constexpr (N == 5) {
        const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
        const float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
        const float2 x0 = v[OFF];
        const float2 a1 = add(v[OFF + S], v[OFF + 4 * S]), b1 = sub(v[OFF + S], v[OFF + 4 * S]);
        const float2 a2 = add(v[OFF + 2 * S], v[OFF + 3 * S]), b2 = sub(v[OFF + 2 * S], v[OFF + 3 * S]);
        const float2 p1 = make_float2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
        const float2 p2 = make_float2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
        const float2 u1 = make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y);
        const float2 u2 = make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y);
        // forward: X1 = p1 - i u1, X4 = p1 + i u1, X2 = p2 - i u2, X3 = p2 + i u2
        const float2 q1 = INV ? make_float2(-u1.y, u1.x) : make_float2(u1.y, -u1.x);
        const float2 q2 = INV ? make_float2(-u2.y, u2.x) : make_float2(u2.y, -u2.x);
        v[OFF] = make_float2(x0.x + a1.x + a2.x, x0.y + a1.y + a2.y);
        v[OFF + S] = add(p1, q1);
        v[OFF + 4 * S] = sub(p1, q1);
        v[OFF + 2 * S] = add(p2, q2);
        v[OFF + 3 * S] = sub(p2, q2);
    } else {
        constexpr int A = first_factor(N), B = N / A;
        static_assert(A < N, "unsupported prime factor in register DFT");
        // step 1: A-point DFTs over n1 (positions n2 + B n1), twiddle W_N^{n2 k1}
        static_for<0, B>([&](auto n2c) {
            constexpr int n2 = decltype(n2c)::value;
            dft<M, A, OFF + S * n2, S * B, INV>(v);
            static_for<1, A>([&](auto k1c) {
                constexpr int k1 = decltype(k1c)::value;
                v[OFF + S * (n2 + B * k1)] = rot<n2 * k1, N, INV>(v[OFF + S * (n2 + B * k1)]);
            });
        });
        // step 2: B-point DFTs over n2 (contiguous run at B k1)
        static_for<0, A>([&](auto k1c) {
            constexpr int k1 = decltype(k1c)::value;
            dft<M, B, OFF + S * B * k1, S, INV>(v);
        });
        // step 3: X[k1 + A k2] sits at position B k1 + k2
        float2 t[N];
#pragma unroll
        for (int i = 0; i < N; ++i) t[i] = v[OFF + S * i];
#pragma unroll
        for (int k1 = 0; k1 < A; ++k1)
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) v[OFF + S * (k1 + A * k2)] = t[B * k1 + k2];
    }
}

// The two-exchange transform of P rings of length N1*N2 in shared memory `buf`
// (ring p at buf + p*LD; natural order in, natural order out).
// twT[k1*N2 + n2] = W_N^{n2 k1} (forward).  Requires blockDim.x == THREADS == P*N1.
template <int N1, int N2, int LD, bool INV>
__device__ __forceinline__ void transform(float2* buf, const float2* __restrict__ twT) {
    constexpr int N = N1 * N2;
    constexpr int P = THREADS / N1;
    static_assert(P * N1 == THREADS, "one phase-B item per thread");
    // phase A
    for (int it = threadIdx.x; it < P * N2; it += THREADS) {
        const int p = it / N2, n2 = it - p * N2;
        float2* r = buf + p * LD + n2;
        float2 a[N1];
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) a[n1] = r[N2 * n1];
        dft<N1, N1, 0, 1, INV>(a);
#pragma unroll
        for (int k1 = 1; k1 < N1; ++k1) {
            float2 w = __ldg(twT + k1 * N2 + n2);
            if (INV) w.y = -w.y;
            a[k1] = make_float2(a[k1].x * w.x - a[k1].y * w.y, a[k1].x * w.y + a[k1].y * w.x);
        }
#pragma unroll
        for (int k1 = 0; k1 < N1; ++k1) r[N2 * k1] = a[k1];
    }
    __syncthreads();
    // phase B
    const int p = threadIdx.x / N1, k1 = threadIdx.x - p * N1;
    float2 b[N2];
    const float2* src = buf + p * LD + N2 * k1;
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) b[n2] = src[n2];
    dft<N2, N2, 0, 1, INV>(b);
    __syncthreads();
    float2* dst = buf + p * LD + k1;
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) dst[N1 * k2] = b[k2];
    __syncthreads();
}

// Phase A for one item given its N1 inputs in registers: DFT, inter-twiddle, write the
// N1 outputs to buf[p*LD + n2 + N2*k1].
template <int N1, int N2, int LD, bool INV>
__device__ __forceinline__ void phase_a_store(float2 (&a)[N1], float2* buf, int p, int n2,
                                              const float2* __restrict__ twT) {
    dft<N1, N1, 0, 1, INV>(a);
#pragma unroll
    for (int k1 = 1; k1 < N1; ++k1) {
        float2 w = __ldg(twT + k1 * N2 + n2);
        if (INV) w.y = -w.y;
        a[k1] = make_float2(a[k1].x * w.x - a[k1].y * w.y, a[k1].x * w.y + a[k1].y * w.x);
    }
    float2* r = buf + p * LD + n2;
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) r[N2 * k1] = a[k1];
}

// Phase B into registers: thread (p, k1) returns X[k1 + N1*k2], k2 < N2, of ring p.
template <int N1, int N2, int LD, bool INV>
__device__ __forceinline__ void phase_b_regs(const float2* buf, float2 (&b)[N2]) {
    const int p = threadIdx.x / N1, k1 = threadIdx.x - p * N1;
    const float2* src = buf + p * LD + N2 * k1;
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) b[n2] = src[n2];
    dft<N2, N2, 0, 1, INV>(b);
}

}  // namespace fft4
}  // namespace sph
