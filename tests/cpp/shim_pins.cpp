// The C++ drop-in (include/sphere_gpu.hpp over libsphgpu.so) run on the GPU against the
// reference itself: every case below calls sphere_gpu:: with the reference's own types
// and checks it against sphere:: (the unmodified reference headers, fp64, in the same
// program) or against the reference tests' analytic known answers
// (proj/tests/test_harmonics.cpp:57-181, test_convolution.cpp:129-261) -- at the fp32 /
// 3xTF32 bar of 1e-5 relative instead of the reference's fp64 1e-10..1e-12.
// Exception pins (CHECK_THROWS_AS in the reference) are kept exactly: the shim rethrows
// SPH_ERR_INVALID_ARGUMENT as std::invalid_argument.
//
// Built by tests/cpp/build.sh (this container, where the reference headers are) into
// tests/cpp/_bin/shim_pins; run by tests/test_cpp_shim_gpu.py on the B200.  Exit code =
// number of failed checks.
#include <cmath>
#include <complex>
#include <cstdio>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "sphere/convolution.hpp"
#include "sphere/field.hpp"
#include "sphere/grid.hpp"
#include "sphere/harmonics.hpp"
#include "sphere_gpu.hpp"

namespace {

int g_fail = 0, g_pass = 0;

void check(bool ok, const std::string& what) {
    if (ok) {
        ++g_pass;
    } else {
        ++g_fail;
        std::printf("FAIL %s\n", what.c_str());
    }
}

template <class Fn>
void check_throws_invalid(Fn fn, const std::string& what) {
    try {
        fn();
    } catch (const std::invalid_argument&) {
        ++g_pass;
        return;
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("FAIL %s: wrong exception type (%s)\n", what.c_str(), e.what());
        return;
    }
    ++g_fail;
    std::printf("FAIL %s: no exception\n", what.c_str());
}

double rel(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / std::max(den, 1e-300));
}
double rel(const std::vector<std::complex<double>>& a, const std::vector<std::complex<double>>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += std::norm(a[i] - b[i]);
        den += std::norm(b[i]);
    }
    return std::sqrt(num / std::max(den, 1e-300));
}

sphere::SphericalField random_field(const sphere::GridSpec& g, size_t c, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    sphere::SphericalField f(g, c);
    for (auto& v : f.data) v = u(rng);
    return f;
}

sphere::SpectralCoeffs random_coeffs(size_t lmax, size_t mmax, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    sphere::SpectralCoeffs c(lmax, mmax, 1);
    for (size_t l = 0; l < lmax; ++l)
        for (size_t m = 0; m <= std::min(l, mmax - 1); ++m) c.at(0, l, m) = {u(rng), m ? u(rng) : 0.0};
    return c;
}

constexpr double kTol = 1e-5;
const double kFourPi = 4.0 * 3.14159265358979323846;

void sht_pins() {
    // test_harmonics.cpp:57-67: a constant hits only uhat_0^0 = sqrt(4 pi)
    {
        const sphere::GridSpec g = sphere::build_gaussian(8, 16);
        sphere::SphericalField f(g, 1);
        for (auto& v : f.data) v = 1.0;
        const sphere::SpectralCoeffs c = sphere_gpu::sht_forward(f, 8, 8);
        double err = 0;
        for (size_t l = 0; l < 8; ++l)
            for (size_t m = 0; m <= l; ++m)
                err = std::max(err, std::abs(c.at(0, l, m) - ((l == 0 && m == 0) ? std::sqrt(kFourPi) : 0.0)));
        check(err <= kTol * std::sqrt(kFourPi), "constant -> uhat_0^0 = sqrt(4 pi)");
    }
    // test_harmonics.cpp:69-79: Re Y_5^3 -> 0.5 at (5, 3), nothing elsewhere
    {
        const sphere::GridSpec g = sphere::build_gaussian(8, 16);
        const sphere::LegendreTable t = sphere::legendre_table(8, 8, g.colatitudes);
        sphere::SphericalField f(g, 1);
        for (size_t i = 0; i < g.nlat; ++i)
            for (size_t j = 0; j < g.nlon; ++j) f.at(0, i, j) = t.at(i, 5, 3) * std::cos(3.0 * g.longitudes[j]);
        const sphere::SpectralCoeffs c = sphere_gpu::sht_forward(f, 8, 8);
        double err = 0;
        for (size_t l = 0; l < 8; ++l)
            for (size_t m = 0; m <= l; ++m)
                err = std::max(err, std::abs(c.at(0, l, m) - ((l == 5 && m == 3) ? std::complex<double>(0.5) : 0.0)));
        check(err <= kTol, "Re Y_5^3 -> 0.5 at (5,3)");
    }
    // test_harmonics.cpp:81-94: Parseval
    {
        const sphere::GridSpec g = sphere::build_gaussian(16, 32);
        const sphere::SphericalField f = sphere_gpu::sht_inverse(random_coeffs(16, 16, 99), g);
        sphere::SphericalField f2(g, 1);
        for (size_t k = 0; k < f.data.size(); ++k) f2.data[k] = f.data[k] * f.data[k];
        const double quad = sphere::integrate(f2)[0];
        const sphere::SpectralCoeffs r = sphere_gpu::sht_forward(f, 16, 16);
        double spec = 0;
        for (size_t l = 0; l < 16; ++l)
            for (size_t m = 0; m <= l; ++m) spec += (m ? 2.0 : 1.0) * std::norm(r.at(0, l, m));
        check(std::abs(spec - quad) <= 2 * kTol * quad, "Parseval");
    }
    // test_harmonics.cpp:96-100: the inverse of zero is zero (exactly)
    {
        const sphere::SphericalField f = sphere_gpu::sht_inverse(sphere::SpectralCoeffs(6, 6), sphere::build_equiangular(9, 16));
        bool zero = true;
        for (double v : f.data) zero = zero && v == 0.0;
        check(zero, "inverse of zero coefficients is zero");
    }
    // test_harmonics.cpp:102-114: equiangular synthesis of Y_2^1, against the reference
    {
        const sphere::GridSpec g = sphere::build_equiangular(9, 16);
        sphere::SpectralCoeffs c(4, 4);
        c.at(0, 2, 1) = {1.0, 0.0};
        check(rel(sphere_gpu::sht_inverse(c, g).data, sphere::sht_inverse(c, g).data) <= kTol,
              "equiangular synthesis of Y_2^1");
    }
    // test_harmonics.cpp:116-131: band-limited round trip on Gaussian 32x64
    {
        const sphere::GridSpec g = sphere::build_gaussian(32, 64);
        const sphere::SpectralCoeffs c = random_coeffs(32, 32, 7);
        const sphere::SphericalField f = sphere_gpu::sht_inverse(c, g);
        const sphere::SpectralCoeffs r = sphere_gpu::sht_forward(f, 32, 32);
        check(rel(r.coeffs, c.coeffs) <= kTol, "Gaussian 32x64 round trip");
    }
    // test_harmonics.cpp:147-161: rotation about the pole = phase e^{-i m dphi}
    {
        const sphere::GridSpec g = sphere::build_gaussian(8, 16);
        const sphere::SpectralCoeffs c = random_coeffs(8, 8, 31);
        const sphere::SphericalField f = sphere_gpu::sht_inverse(c, g);
        sphere::SphericalField fr(g, 1);
        for (size_t i = 0; i < 8; ++i)
            for (size_t j = 0; j < 16; ++j) fr.at(0, i, (j + 3) % 16) = f.at(0, i, j);
        const sphere::SpectralCoeffs cr = sphere_gpu::sht_forward(fr, 8, 8);
        std::vector<std::complex<double>> want(cr.coeffs.size());
        for (size_t l = 0; l < 8; ++l)
            for (size_t m = 0; m < 8; ++m) {
                const double ang = -2.0 * 3.14159265358979323846 * static_cast<double>(m * 3) / 16.0;
                want[l * 8 + m] = c.at(0, l, m) * std::complex<double>(std::cos(ang), std::sin(ang));
            }
        check(rel(cr.coeffs, want) <= kTol, "polar rotation phase");
    }
    // random fields against the reference on both grid kinds (equiangular through the
    // reference's equiangular forward path, dist_sht_forward 1x1 == sht_forward_any_grid)
    {
        const sphere::GridSpec g = sphere::build_gaussian(16, 32);
        const sphere::SphericalField f = random_field(g, 3, 5);
        check(rel(sphere_gpu::sht_forward(f, 16, 16).coeffs, sphere::sht_forward(f, 16, 16).coeffs) <= kTol,
              "Gaussian forward vs reference");
        const sphere::SpectralCoeffs c = sphere::sht_forward(f, 16, 16);
        check(rel(sphere_gpu::sht_inverse(c, g).data, sphere::sht_inverse(c, g).data) <= kTol,
              "Gaussian inverse vs reference");
    }
    // test_harmonics.cpp:174-181: preconditions, incl. the equiangular throw
    {
        const sphere::GridSpec g = sphere::build_gaussian(8, 16);
        sphere::SphericalField f(g, 1);
        check_throws_invalid([&] { (void)sphere_gpu::sht_forward(f, 9, 8); }, "lmax > nlat throws");
        check_throws_invalid([&] { (void)sphere_gpu::sht_forward(f, 8, 9); }, "mmax > nlon/2 throws");
        sphere::SphericalField fe(sphere::build_equiangular(8, 16), 1);
        check_throws_invalid([&] { (void)sphere_gpu::sht_forward(fe, 8, 8); }, "equiangular forward throws");
    }
}

void disco_pins() {
    // test_convolution.cpp:129-163: against the reference operator on three grid pairs
    struct Case {
        sphere::GridSpec gi, go;
        double cut;
        size_t cin, cout;
        const char* name;
    };
    const double pi = 3.14159265358979323846;
    const std::vector<Case> cases = {
        {sphere::build_equiangular(16, 32), sphere::build_equiangular(16, 32), 4 * pi / 16, 3, 2, "eq16 -> eq16"},
        {sphere::build_gaussian(16, 32), sphere::build_gaussian(8, 16), 3 * pi / 8, 3, 2, "ga16 -> ga8"},
        {sphere::build_equiangular(12, 24), sphere::build_equiangular(12, 8), 3 * pi / 12, 1, 1, "eq12 stride 3"},
    };
    for (const Case& k : cases) {
        const sphere::FilterBasis b = sphere::morlet_basis(k.cut);
        const sphere::DiscoOperator rop = sphere::assemble_disco(k.gi, k.go, b);
        const sphere_gpu::DiscoOperator gop = sphere_gpu::assemble_disco(k.gi, k.go, b);
        check(gop.n_basis == rop.n_basis && gop.stride == rop.stride, std::string(k.name) + " operator shape");
        const sphere::SphericalField u = random_field(k.gi, k.cin, 78);
        sphere::MixTensor mix(k.cout, k.cin, rop.n_basis);
        std::mt19937_64 rng(77);
        std::uniform_real_distribution<double> d(-1.0, 1.0);
        for (auto& w : mix.w) w = d(rng);
        check(rel(sphere_gpu::disco_apply(gop, u, mix).data, sphere::disco_apply(rop, u, mix).data) <= kTol,
              std::string(k.name) + " disco_apply vs reference");
        // test_convolution.cpp:214-234: the transpose against the reference's
        const sphere::SphericalField v = random_field(k.go, k.cout, 79);
        check(rel(sphere_gpu::disco_transpose_apply(gop, v, mix).data,
                  sphere::disco_transpose_apply(rop, v, mix).data) <= kTol,
              std::string(k.name) + " disco_transpose_apply vs reference");
    }
    // test_convolution.cpp:247-261: rejects like the reference
    check_throws_invalid(
        [] { (void)sphere_gpu::assemble_disco(sphere::build_gaussian(8, 16), sphere::build_gaussian(4, 8),
                                              sphere::isotropic_basis(1e-4)); },
        "empty support throws");
    check_throws_invalid(
        [] { (void)sphere_gpu::assemble_disco(sphere::build_gaussian(8, 16), sphere::build_gaussian(8, 12),
                                              sphere::isotropic_basis(1.0)); },
        "non-uniform longitude subset throws");
    // spectral_conv (convolution.hpp:286-304) against the reference
    {
        const sphere::GridSpec g = sphere::build_gaussian(16, 32);
        const sphere::SphericalField f = random_field(g, 3, 81);
        sphere::SpectralKernel ker(2, 3, 16);
        std::mt19937_64 rng(82);
        std::uniform_real_distribution<double> d(-1.0, 1.0);
        for (auto& w : ker.k) w = d(rng);
        check(rel(sphere_gpu::spectral_conv(f, ker).data, sphere::spectral_conv(f, ker).data) <= kTol,
              "spectral_conv vs reference");
        sphere::SphericalField fe(sphere::build_equiangular(16, 32), 3);
        check_throws_invalid([&] { (void)sphere_gpu::spectral_conv(fe, ker); }, "spectral_conv equiangular throws");
    }
}

}  // namespace

int main() {
    try {
        sht_pins();
        disco_pins();
    } catch (const std::exception& e) {
        std::printf("FAIL uncaught exception: %s\n", e.what());
        ++g_fail;
    }
    std::printf("shim pins: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
