/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the spherical-operator hot path.
 *
 * A plain-C (C99, fp64, single-threaded) restatement of the reference algorithm
 * (spheretk, /root/reference/proj/include/sphere/ headers).  Every function cites the
 * reference file:line it follows.  It is NOT part of the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and only as
 * the checker.  It is pinned against the reference itself (oracle/_ref/libsphref.so,
 * built from the unmodified headers) through the golden vectors in tests/golden/
 * (tests/test_oracle.py).
 *
 * Conventions (all from the reference):
 *   fields      [C][nlat][nlon] row-major                      field.hpp:15-35
 *   coeffs      [C][lmax][mmax] complex (re,im interleaved),
 *               zero above the diagonal                         harmonics.hpp:24-42
 *   DFT         forward sum x e^{-2 pi i jk/n}, no 1/n          fft.hpp:85-86
 *   mix         [c_out][c_in][K]                                convolution.hpp:126-139
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------ random inputs ---- */

/* proj/tests/oracles.hpp:105-112 random_field: std::mt19937_64(seed) with
 * std::uniform_real_distribution<double>(-1, 1) in storage order.  Restated:
 * MT19937-64 (Matsumoto & Nishimura 2004 parameters, as <random>) and libstdc++'s
 * generate_canonical<double,53> for a 64-bit engine = double(x) / 2^64 (clamped
 * below 1), then a + (b - a) * u. */
void orc_random_uniform(uint64_t seed, size_t n, double* out) {
    enum { NN = 312, MM = 156 };
    const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL,
                   LM = 0x7FFFFFFFULL;
    uint64_t mt[NN];
    size_t mti;
    mt[0] = seed;
    for (mti = 1; mti < NN; mti++)
        mt[mti] = 6364136223846793005ULL * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + mti;
    for (size_t k = 0; k < n; ++k) {
        if (mti >= NN) {
            size_t i;
            uint64_t x;
            for (i = 0; i < NN - MM; i++) {
                x = (mt[i] & UM) | (mt[i + 1] & LM);
                mt[i] = mt[i + MM] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
            }
            for (; i < NN - 1; i++) {
                x = (mt[i] & UM) | (mt[i + 1] & LM);
                mt[i] = mt[i + (MM - NN)] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
            }
            x = (mt[NN - 1] & UM) | (mt[0] & LM);
            mt[NN - 1] = mt[MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
            mti = 0;
        }
        uint64_t x = mt[mti++];
        x ^= (x >> 29) & 0x5555555555555555ULL;
        x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
        x ^= (x << 37) & 0xFFF7EEE000000000ULL;
        x ^= (x >> 43);
        double u = (double)x / 18446744073709551616.0;
        if (u >= 1.0) u = nextafter(1.0, 0.0);
        out[k] = u * 2.0 + (-1.0);
    }
}

/* ---------------------------------------------------------------- grids ---- */

/* grid.hpp:48-63 legendre_pn */
static void legendre_pn(size_t n, double x, double* pn, double* dpn) {
    double p0 = 1.0, p1 = x;
    if (n == 0) { *pn = 1.0; *dpn = 0.0; return; }
    for (size_t k = 2; k <= n; ++k) {
        const double kk = (double)k;
        const double p2 = ((2.0 * kk - 1.0) * x * p1 - (kk - 1.0) * p0) / kk;
        p0 = p1;
        p1 = p2;
    }
    *pn = p1;
    *dpn = (double)n * (x * p1 - p0) / (x * x - 1.0);
}

/* kind 0: equiangular (grid.hpp:69-87), kind 1: Gaussian (grid.hpp:91-128).
 * Returns 0, 1 (invalid argument) or 2 (Newton failure, grid.hpp:117-119). */
int orc_grid(int kind, size_t nlat, size_t nlon, double* colat, double* weights) {
    if (kind == 0) {
        if (nlat < 2 || nlon < 2) return 1;
        const double wfac = 2.0 * ORC_PI * ORC_PI / ((double)nlat * (double)nlon);
        for (size_t i = 0; i < nlat; ++i) {
            colat[i] = ORC_PI * (double)i / (double)nlat;
            weights[i] = wfac * sin(colat[i]);
        }
        return 0;
    }
    if (nlat < 1 || nlon < 2) return 1;
    const double dphi = 2.0 * ORC_PI / (double)nlon;
    for (size_t i = 0; i < nlat; ++i) {
        double x = cos(ORC_PI * ((double)i + 0.75) / ((double)nlat + 0.5));
        double pn = 0.0, dpn = 0.0;
        int converged = 0;
        for (int it = 0; it < 100; ++it) {
            legendre_pn(nlat, x, &pn, &dpn);
            const double dx = pn / dpn;
            x -= dx;
            if (fabs(dx) <= 1e-15) { converged = 1; break; }
        }
        if (!converged) return 2;
        legendre_pn(nlat, x, &pn, &dpn);
        const double wgl = 2.0 / ((1.0 - x * x) * dpn * dpn);
        colat[i] = acos(x);
        weights[i] = wgl * dphi;
    }
    return 0;
}

/* ------------------------------------------------------------------ FFT ---- */
/* complex arrays are interleaved (re, im) doubles */

static int is_pow2(size_t n) { return n > 0 && (n & (n - 1)) == 0; }

/* fft.hpp:22-48 iterative radix-2 with bit reversal */
static void fft_radix2(double* a, size_t n, int inverse) {
    if (n < 2) return;
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double t0 = a[2 * i], t1 = a[2 * i + 1];
            a[2 * i] = a[2 * j]; a[2 * i + 1] = a[2 * j + 1];
            a[2 * j] = t0; a[2 * j + 1] = t1;
        }
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const double ang = (inverse ? 2.0 : -2.0) * ORC_PI / (double)len;
        const double wr0 = cos(ang), wi0 = sin(ang);
        for (size_t i = 0; i < n; i += len) {
            double wr = 1.0, wi = 0.0;
            for (size_t k = 0; k < len / 2; ++k) {
                double* u = a + 2 * (i + k);
                double* v = a + 2 * (i + k + len / 2);
                const double vr = v[0] * wr - v[1] * wi, vi = v[0] * wi + v[1] * wr;
                const double ur = u[0], ui = u[1];
                u[0] = ur + vr; u[1] = ui + vi;
                v[0] = ur - vr; v[1] = ui - vi;
                const double nwr = wr * wr0 - wi * wi0;
                wi = wr * wi0 + wi * wr0;
                wr = nwr;
            }
        }
    }
}

/* fft.hpp:52-83 Bluestein chirp-z over a zero-padded radix-2 FFT of size >= 2n+1 */
static void fft_bluestein(double* a, size_t n, int inverse) {
    size_t m = 1;
    while (m < 2 * n + 1) m <<= 1;
    const double sign = inverse ? 1.0 : -1.0;
    double* chirp = (double*)malloc(sizeof(double) * 2 * n);
    double* x = (double*)calloc(2 * m, sizeof(double));
    double* y = (double*)calloc(2 * m, sizeof(double));
    for (size_t k = 0; k < n; ++k) {
        const size_t k2 = (k * k) % (2 * n);
        const double ang = sign * ORC_PI * (double)k2 / (double)n;
        chirp[2 * k] = cos(ang);
        chirp[2 * k + 1] = sin(ang);
    }
    for (size_t k = 0; k < n; ++k) {
        x[2 * k] = a[2 * k] * chirp[2 * k] - a[2 * k + 1] * chirp[2 * k + 1];
        x[2 * k + 1] = a[2 * k] * chirp[2 * k + 1] + a[2 * k + 1] * chirp[2 * k];
        y[2 * k] = chirp[2 * k];
        y[2 * k + 1] = -chirp[2 * k + 1];
        if (k > 0) { y[2 * (m - k)] = chirp[2 * k]; y[2 * (m - k) + 1] = -chirp[2 * k + 1]; }
    }
    fft_radix2(x, m, 0);
    fft_radix2(y, m, 0);
    for (size_t k = 0; k < m; ++k) {
        const double r = x[2 * k] * y[2 * k] - x[2 * k + 1] * y[2 * k + 1];
        const double i = x[2 * k] * y[2 * k + 1] + x[2 * k + 1] * y[2 * k];
        x[2 * k] = r; x[2 * k + 1] = i;
    }
    fft_radix2(x, m, 1);
    const double scale = 1.0 / (double)m;
    for (size_t k = 0; k < n; ++k) {
        const double xr = x[2 * k] * scale, xi = x[2 * k + 1] * scale;
        a[2 * k] = xr * chirp[2 * k] - xi * chirp[2 * k + 1];
        a[2 * k + 1] = xr * chirp[2 * k + 1] + xi * chirp[2 * k];
    }
    free(chirp); free(x); free(y);
}

/* fft.hpp:87-94 */
void orc_fft(double* a, size_t n, int inverse) {
    if (n == 0) return;
    if (is_pow2(n)) fft_radix2(a, n, inverse);
    else fft_bluestein(a, n, inverse);
}

/* fft.hpp:97-104 rfft_bins: first nbins bins of the forward DFT of a real ring */
void orc_rfft_bins(size_t n, const double* x, size_t nbins, double* out) {
    double* a = (double*)malloc(sizeof(double) * 2 * n);
    for (size_t j = 0; j < n; ++j) { a[2 * j] = x[j]; a[2 * j + 1] = 0.0; }
    orc_fft(a, n, 0);
    memcpy(out, a, sizeof(double) * 2 * nbins);
    free(a);
}

/* ------------------------------------------------------------- Legendre ---- */

/* harmonics.hpp:59-102: Phat_l^m(cos theta_i) into out[n][lmax][mmax] (zero above
 * the diagonal), diagonal seed :73-85, l-recurrence :86-97 */
int orc_legendre_table(size_t lmax, size_t mmax, size_t n, const double* colat, double* out) {
    if (mmax > lmax) return 1;
    memset(out, 0, sizeof(double) * n * lmax * mmax);
    for (size_t i = 0; i < n; ++i) {
        const double x = cos(colat[i]);
        const double omx2 = (1.0 - x) * (1.0 + x);
        double* row = out + i * lmax * mmax;
        for (size_t m = 0; m < mmax; ++m) {
            double pmm = 1.0, fact = 1.0;
            for (size_t k = 1; k <= m; ++k) {
                pmm *= omx2 * fact / (fact + 1.0);
                fact += 2.0;
            }
            pmm = sqrt((2.0 * (double)m + 1.0) * pmm / (4.0 * ORC_PI));
            if (m & 1) pmm = -pmm;
            if (m < lmax) row[m * mmax + m] = pmm;
            if (m + 1 < lmax) {
                const double pmmp1 = x * sqrt(2.0 * (double)m + 3.0) * pmm;
                row[(m + 1) * mmax + m] = pmmp1;
                double oldfact = sqrt(2.0 * (double)m + 3.0);
                double pa = pmm, pb = pmmp1;
                for (size_t l = m + 2; l < lmax; ++l) {
                    const double ld = (double)l, md = (double)m;
                    const double f = sqrt((4.0 * ld * ld - 1.0) / (ld * ld - md * md));
                    const double pl = (x * pb - pa / oldfact) * f;
                    row[l * mmax + m] = pl;
                    oldfact = f;
                    pa = pb;
                    pb = pl;
                }
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ SHT ---- */

/* Forward SHT, any grid kind (the equiangular arithmetic is dist_sht_forward's,
 * distsim.hpp:413-459, which equals harmonics.hpp:136-156 without the kind check
 * at :129-130).  Preconditions harmonics.hpp:131-132. */
int orc_sht_forward(size_t nlat, size_t nlon, const double* colat, const double* weights,
                    size_t lmax, size_t mmax, size_t C, const double* x, double* out) {
    if (mmax > lmax || nlat < lmax || nlon < 2 * mmax || mmax == 0) return 1;
    double* tab = (double*)malloc(sizeof(double) * nlat * lmax * mmax);
    orc_legendre_table(lmax, mmax, nlat, colat, tab);
    const double nlon_over_dphi = (double)nlon / (2.0 * ORC_PI);      /* harmonics.hpp:109 */
    for (size_t i = 0; i < nlat; ++i) {
        const double w = weights[i] * nlon_over_dphi;                  /* harmonics.hpp:111 */
        for (size_t k = 0; k < lmax * mmax; ++k) tab[i * lmax * mmax + k] *= w;
    }
    const double fscale = 2.0 * ORC_PI / (double)nlon;                 /* harmonics.hpp:137 */
    double* G = (double*)malloc(sizeof(double) * 2 * nlat * mmax);
    double* ring = (double*)malloc(sizeof(double) * 2 * mmax);
    for (size_t c = 0; c < C; ++c) {
        for (size_t i = 0; i < nlat; ++i) {
            orc_rfft_bins(nlon, x + (c * nlat + i) * nlon, mmax, ring);
            for (size_t m = 0; m < mmax; ++m) {
                G[2 * (i * mmax + m)] = ring[2 * m] * fscale;
                G[2 * (i * mmax + m) + 1] = ring[2 * m + 1] * fscale;
            }
        }
        double* o = out + 2 * c * lmax * mmax;
        memset(o, 0, sizeof(double) * 2 * lmax * mmax);
        for (size_t l = 0; l < lmax; ++l) {                            /* harmonics.hpp:147-154 */
            const size_t mtop = l < mmax - 1 ? l : mmax - 1;
            for (size_t m = 0; m <= mtop; ++m) {
                double ar = 0.0, ai = 0.0;
                for (size_t i = 0; i < nlat; ++i) {
                    const double t = tab[(i * lmax + l) * mmax + m];
                    ar += t * G[2 * (i * mmax + m)];
                    ai += t * G[2 * (i * mmax + m) + 1];
                }
                o[2 * (l * mmax + m)] = ar;
                o[2 * (l * mmax + m) + 1] = ai;
            }
        }
    }
    free(tab); free(G); free(ring);
    return 0;
}

/* Inverse SHT, any grid (harmonics.hpp:173-200): per ring, Legendre synthesis for
 * m < msynth = min(mmax, (nlon-1)/2+1) then real part of the inverse DFT. */
int orc_sht_inverse(size_t nlat, size_t nlon, const double* colat, size_t lmax, size_t mmax,
                    size_t C, const double* coeffs, double* out) {
    if (mmax > lmax) return 1;
    double* tab = (double*)malloc(sizeof(double) * nlat * lmax * mmax);
    orc_legendre_table(lmax, mmax, nlat, colat, tab);
    const size_t msynth = mmax < (nlon - 1) / 2 + 1 ? mmax : (nlon - 1) / 2 + 1;
    double* bins = (double*)malloc(sizeof(double) * 2 * nlon);
    for (size_t c = 0; c < C; ++c) {
        const double* cf = coeffs + 2 * c * lmax * mmax;
        for (size_t i = 0; i < nlat; ++i) {
            memset(bins, 0, sizeof(double) * 2 * nlon);
            for (size_t m = 0; m < msynth; ++m) {
                double hr = 0.0, hi = 0.0;
                for (size_t l = m; l < lmax; ++l) {
                    const double t = tab[(i * lmax + l) * mmax + m];
                    hr += cf[2 * (l * mmax + m)] * t;
                    hi += cf[2 * (l * mmax + m) + 1] * t;
                }
                bins[2 * m] = hr;
                bins[2 * m + 1] = hi;
                if (m > 0) { bins[2 * (nlon - m)] = hr; bins[2 * (nlon - m) + 1] = -hi; }
            }
            orc_fft(bins, nlon, 1);                                    /* fft.hpp:108-113 */
            for (size_t j = 0; j < nlon; ++j) out[(c * nlat + i) * nlon + j] = bins[2 * j];
        }
    }
    free(tab); free(bins);
    return 0;
}

/* ---------------------------------------------------------------- DISCO ---- */

/* convolution.hpp:38-55 FilterBasis::eval (complex), :58-68 eval_real.
 * pairs: (l_w, m_w) list; k enumerates real parts then imaginary parts per pair,
 * (0,0) contributes only its real part. */
static double basis_eval_real(const int* pairs, size_t npairs, double cutoff, size_t k,
                              double theta, double phi) {
    size_t b = 0;
    for (; b < npairs; ++b) {
        const size_t parts = (pairs[2 * b] == 0 && pairs[2 * b + 1] == 0) ? 1 : 2;
        if (k < parts) break;
        k -= parts;
    }
    const double tp = theta / cutoff;
    if (tp > 1.0) return 0.0;
    const double c = cos(0.5 * ORC_PI * tp);
    const double h = c * c;
    const double arg = ORC_PI * tp * ((double)pairs[2 * b] * sin(phi) +
                                      (double)pairs[2 * b + 1] * cos(phi));
    return k == 0 ? h * cos(arg) : h * sin(arg);
}

size_t orc_basis_nreal(const int* pairs, size_t npairs) {
    size_t n = 0;
    for (size_t b = 0; b < npairs; ++b) n += (pairs[2 * b] == 0 && pairs[2 * b + 1] == 0) ? 1 : 2;
    return n;
}

/* convolution.hpp:93-101 chart_coordinates (distance, azimuth from the southward meridian) */
static void chart(double theta_out, double theta_in, double dphi, double* dist, double* az) {
    const double st_o = sin(theta_out), ct_o = cos(theta_out);
    const double st_i = sin(theta_in), ct_i = cos(theta_in);
    const double cd = cos(dphi);
    const double x = ct_o * st_i * cd - st_o * ct_i;
    const double y = st_i * sin(dphi);
    const double z = st_o * st_i * cd + ct_o * ct_i;
    *dist = atan2(hypot(x, y), z);
    *az = atan2(y, x);
}

/* convolution.hpp:141-177 assemble_disco, in a CSR layout that keeps the
 * reference's entry order: row h_out holds entries [row_ptr[h], row_ptr[h+1]),
 * each with (h_in, w_rel) shared by all K basis functions and vals[e*K + k] =
 * b_k * w_in (the reference `value`), base[e*K + k] = b_k.
 * Call with h_in == NULL to only count (row_ptr filled).  Returns 0, 1 on
 * incompatible longitudes (:143-145) or 3 on an empty support row (:172-174). */
int orc_disco_assemble(size_t in_nlat, size_t in_nlon, const double* in_colat,
                       const double* in_w, size_t out_nlat, size_t out_nlon,
                       const double* out_colat, const int* pairs, size_t npairs, double cutoff,
                       int64_t* row_ptr, int32_t* h_in, int32_t* w_rel, double* vals,
                       double* base) {
    if (out_nlon == 0 || in_nlon % out_nlon != 0) return 1;
    const size_t K = orc_basis_nreal(pairs, npairs);
    int64_t n = 0;
    row_ptr[0] = 0;
    for (size_t h = 0; h < out_nlat; ++h) {
        const double theta_out = out_colat[h];
        size_t support = 0;
        for (size_t hi = 0; hi < in_nlat; ++hi) {
            const double theta_in = in_colat[hi];
            if (fabs(theta_in - theta_out) >= cutoff) continue;      /* :159 */
            const double w_in = in_w[hi];
            for (size_t wj = 0; wj < in_nlon; ++wj) {
                const double lon = 2.0 * ORC_PI * (double)wj / (double)in_nlon;  /* grid.hpp:126 */
                double dist, az;
                chart(theta_out, theta_in, lon, &dist, &az);
                if (dist >= cutoff) continue;                          /* :164 strict */
                ++support;
                if (h_in) {
                    h_in[n] = (int32_t)hi;
                    w_rel[n] = (int32_t)wj;
                    for (size_t k = 0; k < K; ++k) {
                        const double b = basis_eval_real(pairs, npairs, cutoff, k, dist, az);
                        vals[n * K + k] = b * w_in;
                        base[n * K + k] = b;
                    }
                }
                ++n;
            }
        }
        if (support == 0) return 3;
        row_ptr[h + 1] = n;
    }
    return 0;
}

/* convolution.hpp:181-220 disco_apply: gather t[k][c][h][w] (:192-205) then the
 * channel mix y[o] += mix[o][c][k] t[k][c] (:207-218, zero weights skipped). */
void orc_disco_apply(size_t in_nlat, size_t in_nlon, size_t out_nlat, size_t out_nlon, size_t K,
                     const int64_t* row_ptr, const int32_t* h_in, const int32_t* w_rel,
                     const double* vals, size_t cin, size_t cout, const double* x,
                     const double* mix, double* y) {
    const size_t stride = in_nlon / out_nlon;
    const size_t plane = out_nlat * out_nlon;
    double* t = (double*)calloc(K * cin * plane, sizeof(double));
    for (size_t k = 0; k < K; ++k)
        for (size_t h = 0; h < out_nlat; ++h)
            for (int64_t e = row_ptr[h]; e < row_ptr[h + 1]; ++e)
                for (size_t c = 0; c < cin; ++c) {
                    const double* u = x + (c * in_nlat + (size_t)h_in[e]) * in_nlon;
                    double* dst = t + ((k * cin + c) * out_nlat + h) * out_nlon;
                    const double v = vals[e * K + k];
                    size_t col = (size_t)w_rel[e];
                    for (size_t w = 0; w < out_nlon; ++w) {
                        dst[w] += v * u[col];
                        col += stride;
                        if (col >= in_nlon) col -= in_nlon;
                    }
                }
    memset(y, 0, sizeof(double) * cout * plane);
    for (size_t o = 0; o < cout; ++o)
        for (size_t c = 0; c < cin; ++c)
            for (size_t k = 0; k < K; ++k) {
                const double wkc = mix[(o * cin + c) * K + k];
                if (wkc == 0.0) continue;
                const double* src = t + (k * cin + c) * plane;
                double* yo = y + o * plane;
                for (size_t p = 0; p < plane; ++p) yo[p] += wkc * src[p];
            }
    free(t);
}

/* convolution.hpp:226-266 disco_transpose_apply: x on the output grid (cout
 * channels) -> y on the input grid (cin channels); entries re-weighted with the
 * output-grid weight (base * w_out, :258). */
void orc_disco_transpose_apply(size_t in_nlat, size_t in_nlon, size_t out_nlat, size_t out_nlon,
                               const double* out_w, size_t K, const int64_t* row_ptr,
                               const int32_t* h_in, const int32_t* w_rel, const double* base,
                               size_t cin, size_t cout, const double* x, const double* mix,
                               double* y) {
    const size_t stride = in_nlon / out_nlon;
    double* vrow = (double*)malloc(sizeof(double) * out_nlon);
    memset(y, 0, sizeof(double) * cin * in_nlat * in_nlon);
    for (size_t k = 0; k < K; ++k)
        for (size_t h = 0; h < out_nlat; ++h) {
            const double w_out = out_w[h];
            for (size_t ci = 0; ci < cin; ++ci) {
                memset(vrow, 0, sizeof(double) * out_nlon);
                for (size_t co = 0; co < cout; ++co) {
                    const double wkc = mix[(co * cin + ci) * K + k];
                    if (wkc == 0.0) continue;
                    const double* v = x + (co * out_nlat + h) * out_nlon;
                    for (size_t w = 0; w < out_nlon; ++w) vrow[w] += wkc * v[w];
                }
                for (int64_t e = row_ptr[h]; e < row_ptr[h + 1]; ++e) {
                    const double scale = base[e * K + k] * w_out;
                    double* dst = y + (ci * in_nlat + (size_t)h_in[e]) * in_nlon;
                    size_t col = (size_t)w_rel[e];
                    for (size_t w = 0; w < out_nlon; ++w) {
                        dst[col] += scale * vrow[w];
                        col += stride;
                        if (col >= in_nlon) col -= in_nlon;
                    }
                }
            }
        }
    free(vrow);
}

/* ------------------------------------------------------- spectral conv ---- */

/* convolution.hpp:286-304 (the Gaussian-only check :287-288 is the caller's):
 * lmax = min(klmax, nlat), mmax = min(lmax, nlon/2); forward SHT, then
 * y(o,l,m) = sum_i c(i,l,m) k(o,i,l) for m <= min(l, mmax-1), inverse SHT. */
int orc_spectral_conv(size_t nlat, size_t nlon, const double* colat, const double* weights,
                      size_t cin, size_t cout, size_t klmax, const double* kernel,
                      const double* x, double* y) {
    const size_t lmax = klmax < nlat ? klmax : nlat;
    const size_t mmax = lmax < nlon / 2 ? lmax : nlon / 2;
    double* c = (double*)malloc(sizeof(double) * 2 * cin * lmax * mmax);
    double* o = (double*)calloc(2 * cout * lmax * mmax, sizeof(double));
    int rc = orc_sht_forward(nlat, nlon, colat, weights, lmax, mmax, cin, x, c);
    if (rc) { free(c); free(o); return rc; }
    for (size_t oc = 0; oc < cout; ++oc)
        for (size_t i = 0; i < cin; ++i)
            for (size_t l = 0; l < lmax; ++l) {
                const double kl = kernel[(oc * cin + i) * klmax + l];
                if (kl == 0.0) continue;
                const size_t mtop = l < mmax - 1 ? l : mmax - 1;
                for (size_t m = 0; m <= mtop; ++m) {
                    o[2 * ((oc * lmax + l) * mmax + m)] += c[2 * ((i * lmax + l) * mmax + m)] * kl;
                    o[2 * ((oc * lmax + l) * mmax + m) + 1] +=
                        c[2 * ((i * lmax + l) * mmax + m) + 1] * kl;
                }
            }
    rc = orc_sht_inverse(nlat, nlon, colat, lmax, mmax, cout, o, y);
    free(c); free(o);
    return rc;
}

/* ---------------------------------------------------------- block MLP ---- */

/* model.hpp:42-44 exact-erfc GeLU */
double orc_gelu(double x) { return x * 0.5 * erfc(-x / sqrt(2.0)); }

/* model.hpp:355-368: out = x + scales .* (W2 gelu(W1 gelu(conv) + b1) + b2) per point;
 * conv [C][npts], x/out [C][npts], w1 [H][C], w2 [C][H]. */
void orc_block_epilogue(size_t C, size_t H, size_t npts, const double* conv, const double* x,
                        const double* w1, const double* b1, const double* w2, const double* b2,
                        const double* scales, double* out) {
    double* g = (double*)malloc(sizeof(double) * C);
    double* h = (double*)malloc(sizeof(double) * H);
    memcpy(out, x, sizeof(double) * C * npts);
    for (size_t p = 0; p < npts; ++p) {
        for (size_t ch = 0; ch < C; ++ch) g[ch] = orc_gelu(conv[ch * npts + p]);
        for (size_t i = 0; i < H; ++i) {
            double acc = b1[i];
            for (size_t ch = 0; ch < C; ++ch) acc += w1[i * C + ch] * g[ch];
            h[i] = orc_gelu(acc);
        }
        for (size_t ch = 0; ch < C; ++ch) {
            double acc = b2[ch];
            for (size_t i = 0; i < H; ++i) acc += w2[ch * H + i] * h[i];
            out[ch * npts + p] += scales[ch] * acc;
        }
    }
    free(g); free(h);
}
