// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI driver around the UNMODIFIED reference headers (spheretk, header-only
// C++20 fp64).  Built by oracle/build_ref.sh from /root/reference/proj/include
// into oracle/_ref/libsphref.so (git-ignored).  Used to
//   * generate the golden vectors under tests/golden/ (tests/golden/make_golden.py),
//   * pin the C restatement in oracle/sphere_oracle.c against the reference itself,
//   * time the reference CPU path on the GPU box's host cores (bench.py
//     --impl reference / cpu_baseline, kind "reference").
// No reference source is copied: every function below calls the reference's own
// public API (namespace sphere) on caller-provided buffers.

#include <atomic>
#include <random>
#include <chrono>
#include <complex>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sphere/convolution.hpp"
#include "sphere/resample.hpp"
#include "sphere/sfd.hpp"
#include "sphere/noise.hpp"
#include "sphere/loss.hpp"
#include "sphere/metrics.hpp"
#include "sphere/distsim.hpp"
#include "sphere/grid.hpp"
#include "sphere/harmonics.hpp"
#include "sphere/model.hpp"

using namespace sphere;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

GridSpec make_grid(int kind, size_t nlat, size_t nlon) {
    return kind == 0 ? build_equiangular(nlat, nlon) : build_gaussian(nlat, nlon);
}

SphericalField make_field(const GridSpec& g, size_t c, const double* x) {
    SphericalField f(g, c);
    if (x) std::memcpy(f.data.data(), x, sizeof(double) * f.data.size());
    return f;
}

void put_coeffs(const SpectralCoeffs& c, double* out) {
    for (size_t i = 0; i < c.coeffs.size(); ++i) {
        out[2 * i] = c.coeffs[i].real();
        out[2 * i + 1] = c.coeffs[i].imag();
    }
}

SpectralCoeffs get_coeffs(size_t lmax, size_t mmax, size_t ch, const double* in) {
    SpectralCoeffs c(lmax, mmax, ch);
    for (size_t i = 0; i < c.coeffs.size(); ++i) c.coeffs[i] = {in[2 * i], in[2 * i + 1]};
    return c;
}

FilterBasis make_basis(int basis, double cutoff) {
    return basis == 0 ? morlet_basis(cutoff) : isotropic_basis(cutoff);
}

MixTensor make_mix(size_t co, size_t ci, size_t k, const double* w) {
    MixTensor m(co, ci, k);
    std::memcpy(m.w.data(), w, sizeof(double) * m.w.size());
    return m;
}

NdArray<double> as_tensor(const SphericalField& f) {
    return NdArray<double>({f.channels, f.grid.nlat, f.grid.nlon}, f.data);
}

void put_csv(const TrafficLog& log, char* csv, size_t cap) {
    if (!csv || cap == 0) return;
    const std::string s = log.csv();
    std::snprintf(csv, cap, "%s", s.c_str());
}
}  // namespace

#define REF_TRY try {
#define REF_CATCH                                                         \
    }                                                                     \
    catch (const std::invalid_argument& e) { return fail(e, 1); }         \
    catch (const std::runtime_error& e) { return fail(e, 2); }            \
    catch (const std::exception& e) { return fail(e, 3); }                \
    return 0;

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// proj/tests/oracles.hpp:105-112 random_field semantics: mt19937_64(seed) and
// uniform_real_distribution<double>(-1, 1), drawn in storage order.
void ref_random_uniform(unsigned long long seed, size_t n, double* out) {
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (size_t i = 0; i < n; ++i) out[i] = u(gen);
}

// grid.hpp:69 / :91
int ref_grid(int kind, size_t nlat, size_t nlon, double* colat, double* weights) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    std::memcpy(colat, g.colatitudes.data(), sizeof(double) * nlat);
    std::memcpy(weights, g.quad_weights.data(), sizeof(double) * nlat);
    REF_CATCH
}

// harmonics.hpp:59 (weighted=0) / :106 (weighted=1, needs the grid)
int ref_legendre_table(size_t lmax, size_t mmax, int kind, size_t nlat, size_t nlon,
                       int weighted, double* out) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    const LegendreTable t = weighted ? weighted_legendre_table(lmax, mmax, g)
                                     : legendre_table(lmax, mmax, g.colatitudes);
    std::memcpy(out, t.values.data(), sizeof(double) * t.values.size());
    REF_CATCH
}

// fft.hpp:97 rfft_bins (forward, no 1/n)
int ref_rfft_bins(size_t n, const double* x, size_t nbins, double* out) {
    REF_TRY
    const auto b = rfft_bins(std::span<const double>(x, n), nbins);
    for (size_t k = 0; k < nbins; ++k) {
        out[2 * k] = b[k].real();
        out[2 * k + 1] = b[k].imag();
    }
    REF_CATCH
}

// Forward SHT.  path 0: serial sphere::sht_forward (harmonics.hpp:159, Gaussian only,
// throws on equiangular exactly like the reference).  path 1: dist_sht_forward with
// CommGrid(1,1,1,1) (distsim.hpp:404), the reference's only equiangular forward.
int ref_sht_forward(int kind, size_t nlat, size_t nlon, size_t lmax, size_t mmax, size_t ch,
                    const double* x, double* out, int path) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    const SphericalField f = make_field(g, ch, x);
    if (path == 0) {
        put_coeffs(sht_forward(f, lmax, mmax), out);
    } else {
        DistContext ctx{CommGrid(1, 1, 1, 1), {}};
        auto views = shard(ctx, std::vector<NdArray<double>>{as_tensor(f)},
                           {{1, CommAxis::polar}, {2, CommAxis::azimuth}});
        auto res = dist_sht_forward(ctx, views, g, lmax, mmax);
        const auto glob = unshard(ctx, res, {{1, CommAxis::polar}, {2, CommAxis::azimuth}});
        for (size_t i = 0; i < glob.data.size(); ++i) {
            out[2 * i] = glob.data[i].real();
            out[2 * i + 1] = glob.data[i].imag();
        }
    }
    REF_CATCH
}

// harmonics.hpp:202
int ref_sht_inverse(int kind, size_t nlat, size_t nlon, size_t lmax, size_t mmax, size_t ch,
                    const double* coeffs, double* out) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    const SphericalField f = sht_inverse(get_coeffs(lmax, mmax, ch, coeffs), g);
    std::memcpy(out, f.data.data(), sizeof(double) * f.data.size());
    REF_CATCH
}

// convolution.hpp:141 -- structural summary of the assembled operator:
// rows[h_out] = support size (entries per basis function), plus total nnz.
int ref_disco_rows(int in_kind, size_t in_nlat, size_t in_nlon, int out_kind, size_t out_nlat,
                   size_t out_nlon, int basis, double cutoff, size_t* row_nnz, size_t* n_basis) {
    REF_TRY
    const DiscoOperator op = assemble_disco(make_grid(in_kind, in_nlat, in_nlon),
                                            make_grid(out_kind, out_nlat, out_nlon),
                                            make_basis(basis, cutoff));
    *n_basis = op.n_basis;
    for (size_t h = 0; h < out_nlat; ++h) row_nnz[h] = op.rows[0][h].size();
    REF_CATCH
}

// Dump the assembled entries: for every (k, h_out) row, entries in order.
// h_in/w_rel are int64, values/base double; caller sizes buffers from ref_disco_rows.
int ref_disco_entries(int in_kind, size_t in_nlat, size_t in_nlon, int out_kind,
                      size_t out_nlat, size_t out_nlon, int basis, double cutoff,
                      long long* h_in, long long* w_rel, double* value, double* base) {
    REF_TRY
    const DiscoOperator op = assemble_disco(make_grid(in_kind, in_nlat, in_nlon),
                                            make_grid(out_kind, out_nlat, out_nlon),
                                            make_basis(basis, cutoff));
    size_t n = 0;
    for (size_t k = 0; k < op.n_basis; ++k)
        for (size_t h = 0; h < out_nlat; ++h)
            for (const DiscoEntry& e : op.rows[k][h]) {
                h_in[n] = static_cast<long long>(e.h_in);
                w_rel[n] = static_cast<long long>(e.w_rel);
                value[n] = e.value;
                base[n] = e.base;
                ++n;
            }
    REF_CATCH
}

// convolution.hpp:181
int ref_disco_apply(int in_kind, size_t in_nlat, size_t in_nlon, int out_kind, size_t out_nlat,
                    size_t out_nlon, int basis, double cutoff, size_t cin, size_t cout,
                    const double* x, const double* mix, double* y) {
    REF_TRY
    const GridSpec gi = make_grid(in_kind, in_nlat, in_nlon);
    const DiscoOperator op =
        assemble_disco(gi, make_grid(out_kind, out_nlat, out_nlon), make_basis(basis, cutoff));
    const SphericalField out =
        disco_apply(op, make_field(gi, cin, x), make_mix(cout, cin, op.n_basis, mix));
    std::memcpy(y, out.data.data(), sizeof(double) * out.data.size());
    REF_CATCH
}

// convolution.hpp:226 ; x lives on the OUTPUT grid with cout channels, y on the input grid.
int ref_disco_transpose_apply(int in_kind, size_t in_nlat, size_t in_nlon, int out_kind,
                              size_t out_nlat, size_t out_nlon, int basis, double cutoff,
                              size_t cin, size_t cout, const double* x, const double* mix,
                              double* y) {
    REF_TRY
    const GridSpec go = make_grid(out_kind, out_nlat, out_nlon);
    const DiscoOperator op =
        assemble_disco(make_grid(in_kind, in_nlat, in_nlon), go, make_basis(basis, cutoff));
    const SphericalField out = disco_transpose_apply(op, make_field(go, cout, x),
                                                     make_mix(cout, cin, op.n_basis, mix));
    std::memcpy(y, out.data.data(), sizeof(double) * out.data.size());
    REF_CATCH
}

// resample.hpp:66-114 bilinear_resample (with the pole extension of :20-62);
// in_last_pi = 1 sets the input grid's last colatitude to pi (test_resample.cpp:46-47)
int ref_bilinear_resample(int in_kind, size_t in_nlat, size_t in_nlon, int in_last_pi, int out_kind,
                          size_t out_nlat, size_t out_nlon, size_t C, const double* x, double* y) {
    REF_TRY
    GridSpec gi = make_grid(in_kind, in_nlat, in_nlon);
    if (in_last_pi) gi.colatitudes.back() = pi;
    const GridSpec go = make_grid(out_kind, out_nlat, out_nlon);
    const SphericalField out = bilinear_resample(make_field(gi, C, x), go);
    std::memcpy(y, out.data.data(), sizeof(double) * out.data.size());
    REF_CATCH
}

// resample.hpp:120-132 spectral_resample -> y [C][out_nlat][out_nlon]
int ref_spectral_resample(int in_kind, size_t in_nlat, size_t in_nlon, int out_kind, size_t out_nlat,
                          size_t out_nlon, size_t C, const double* x, double* y) {
    REF_TRY
    const GridSpec gi = make_grid(in_kind, in_nlat, in_nlon);
    const GridSpec go = make_grid(out_kind, out_nlat, out_nlon);
    const SphericalField out = spectral_resample(make_field(gi, C, x), go);
    std::memcpy(y, out.data.data(), sizeof(double) * out.data.size());
    REF_CATCH
}

// metrics.hpp:300-314 angular_psd -> psd [C][nlat]
int ref_angular_psd(int kind, size_t nlat, size_t nlon, size_t C, const double* x, double* psd) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    const auto out = angular_psd(make_field(g, C, x));
    for (size_t c = 0; c < C; ++c) std::memcpy(psd + c * nlat, out[c].data(), sizeof(double) * nlat);
    REF_CATCH
}

// loss.hpp:37-81 spectral_crps_loss; ens [E][C][H][W], obs [C][H][W]; variant 0 cdf,
// 1 spread_skill, 2 fair -> out [C]
int ref_spectral_crps_loss(int kind, size_t nlat, size_t nlon, size_t E, size_t C, const double* ens,
                           const double* obs, size_t lmax_sum, int variant, double* out) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    EnsembleField ef(g, E, C);
    std::memcpy(ef.values.data(), ens, sizeof(double) * ef.values.size());
    const auto r = spectral_crps_loss(ef, make_field(g, C, obs), lmax_sum, static_cast<CrpsVariant>(variant));
    std::memcpy(out, r.data(), sizeof(double) * C);
    REF_CATCH
}

// noise.hpp:95-97 + :113-140: `steps` steps of a NoiseStream (lambda = sigma = 1, the
// given k_T per channel) -> the final synthesized field [C][H][W] and the channels'
// spectral states [C][lmax][lmax] complex (interleaved re/im)
int ref_noise_stream(int kind, size_t nlat, size_t nlon, size_t lmax, size_t C, const double* kts,
                     uint64_t seed, size_t steps, double* field, double* coeffs) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    std::vector<DiffusionParams> ps;
    for (size_t c = 0; c < C; ++c) ps.push_back(diffusion_params(1.0, 1.0, kts[c], lmax));
    Rng rng(seed);
    std::vector<NoiseState> st;
    for (auto& p : ps) st.push_back(make_noise_state(p));
    for (size_t s = 0; s < steps; ++s)
        for (size_t c = 0; c < C; ++c) st[c] = diffusion_step(st[c], ps[c], rng);
    for (size_t c = 0; c < C; ++c) {
        const SphericalField f = noise_field(st[c], g);
        std::memcpy(field + c * f.npoints(), f.data.data(), sizeof(double) * f.npoints());
        for (size_t l = 0; l < lmax; ++l)
            for (size_t m = 0; m < lmax; ++m) {
                const std::complex<double> v = st[c].coeffs.at(0, l, m);
                coeffs[((c * lmax + l) * lmax + m) * 2] = v.real();
                coeffs[((c * lmax + l) * lmax + m) * 2 + 1] = v.imag();
            }
    }
    REF_CATCH
}

// sfd.hpp:107-131 write_sfd (default channel names) and :183-206 write_weights of two
// tensors ("w1" [a][b], "b1" [a]) with meta {"model": "fcn3", "version": 3}
int ref_write_sfd(const char* path, int kind, size_t nlat, size_t nlon, size_t C, const double* data) {
    REF_TRY
    write_sfd(path, make_field(make_grid(kind, nlat, nlon), C, data));
    REF_CATCH
}

int ref_write_weights(const char* path, size_t a, size_t b, const double* w1, const double* b1) {
    REF_TRY
    NamedTensor t1{"w1", {a, b}, std::vector<double>(w1, w1 + a * b)};
    NamedTensor t2{"b1", {a}, std::vector<double>(b1, b1 + a)};
    write_weights(path, {t1, t2}, nlohmann::json{{"model", "fcn3"}, {"version", 3}});
    REF_CATCH
}

// read back through the reference readers: returns the io error code + 1 on IoError
int ref_read_sfd(const char* path, double* data, size_t cap, size_t* C, size_t* nlat, size_t* nlon) {
    try {
        const SfdContents c = read_sfd(path);
        *C = c.field.channels;
        *nlat = c.field.grid.nlat;
        *nlon = c.field.grid.nlon;
        if (c.field.data.size() <= cap) std::memcpy(data, c.field.data.data(), 8 * c.field.data.size());
        return 0;
    } catch (const IoError& e) {
        return 1 + static_cast<int>(e.code());
    }
}

// metrics.hpp:212-231 crps_field (the serial target of dist_crps, test_distsim.cpp:250-275)
int ref_crps_field(int kind, size_t nlat, size_t nlon, size_t E, size_t C, const double* ens,
                   const double* obs, int variant, double* out) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    EnsembleField ef(g, E, C);
    std::memcpy(ef.values.data(), ens, sizeof(double) * ef.values.size());
    const auto r = crps_field(ef, make_field(g, C, obs), g, static_cast<CrpsVariant>(variant));
    std::memcpy(out, r.data(), sizeof(double) * C);
    REF_CATCH
}

// convolution.hpp:286 (Gaussian only)
int ref_spectral_conv(int kind, size_t nlat, size_t nlon, size_t cin, size_t cout, size_t klmax,
                      const double* kernel, const double* x, double* y) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    SpectralKernel k(cout, cin, klmax);
    std::memcpy(k.k.data(), kernel, sizeof(double) * k.k.size());
    const SphericalField out = spectral_conv(make_field(g, cin, x), k);
    std::memcpy(y, out.data.data(), sizeof(double) * out.data.size());
    REF_CATCH
}

// model.hpp:337 block_apply with a hand-built Model: latent grid Gaussian(nlat,nlon),
// latent channels C = (levels+1)*embed_group, cond channels = embed_group.
// global != 0 -> spectral_conv with kernel [C][C+Cc][klmax]; else disco with mix
// [C][C+Cc][K] and block_op = assemble_disco(latent, latent, morlet(cutoff)).
int ref_block_apply(size_t nlat, size_t nlon, size_t levels, size_t embed_group, size_t hidden,
                    int global, double cutoff, size_t klmax, const double* x, const double* cond,
                    const double* conv_w, const double* w1, const double* b1, const double* w2,
                    const double* b2, const double* scales, double* y) {
    REF_TRY
    Model m;
    ModelConfig& c = m.config;
    c.latent_grid = build_gaussian(nlat, nlon);
    c.in_grid = c.latent_grid;
    c.out_grid = c.latent_grid;
    c.atmo_levels = levels;
    c.atmo_vars = 1;
    c.surface_channels = 1;
    c.aux_channels = 1;
    c.noise_channels = 1;
    c.embed_group = embed_group;
    c.mlp_hidden = hidden;
    c.theta_cutoff = cutoff;
    const size_t C = c.latent_state_channels();
    const size_t Cc = c.latent_cond_channels();
    BlockWeights bw;
    bw.global = global != 0;
    if (bw.global) {
        bw.kernel = SpectralKernel(C, C + Cc, klmax);
        std::memcpy(bw.kernel.k.data(), conv_w, sizeof(double) * bw.kernel.k.size());
    } else {
        m.block_op = assemble_disco(c.latent_grid, c.latent_grid, morlet_basis(cutoff));
        bw.mix = make_mix(C, C + Cc, m.block_op.n_basis, conv_w);
    }
    bw.w1.assign(w1, w1 + hidden * C);
    bw.b1.assign(b1, b1 + hidden);
    bw.w2.assign(w2, w2 + C * hidden);
    bw.b2.assign(b2, b2 + C);
    bw.scales.assign(scales, scales + C);
    m.blocks.push_back(std::move(bw));
    const SphericalField out =
        block_apply(m, 0, make_field(c.latent_grid, C, x), make_field(c.latent_grid, Cc, cond));
    std::memcpy(y, out.data.data(), sizeof(double) * out.data.size());
    REF_CATCH
}

size_t ref_block_channels(size_t levels, size_t embed_group) {
    return (levels + 1) * embed_group;
}

// distsim.hpp:404 on a CommGrid(1,1,nh,nw); output unsharded [C][lmax][mmax] complex.
int ref_dist_sht_forward(int kind, size_t nlat, size_t nlon, size_t lmax, size_t mmax, size_t ch,
                         size_t nh, size_t nw, const double* x, double* out, char* csv,
                         size_t csv_cap) {
    REF_TRY
    const GridSpec g = make_grid(kind, nlat, nlon);
    const SphericalField f = make_field(g, ch, x);
    DistContext ctx{CommGrid(1, 1, nh, nw), {}};
    auto views = shard(ctx, std::vector<NdArray<double>>{as_tensor(f)},
                       {{1, CommAxis::polar}, {2, CommAxis::azimuth}});
    auto res = dist_sht_forward(ctx, views, g, lmax, mmax);
    const auto glob = unshard(ctx, res, {{1, CommAxis::polar}, {2, CommAxis::azimuth}});
    for (size_t i = 0; i < glob.data.size(); ++i) {
        out[2 * i] = glob.data[i].real();
        out[2 * i + 1] = glob.data[i].imag();
    }
    put_csv(ctx.log, csv, csv_cap);
    REF_CATCH
}

// distsim.hpp:468 on a CommGrid(1,1,nh,nw); output unsharded [cout][nlat_out][nlon_out].
int ref_dist_disco_apply(int in_kind, size_t in_nlat, size_t in_nlon, int out_kind,
                         size_t out_nlat, size_t out_nlon, int basis, double cutoff, size_t cin,
                         size_t cout, size_t nh, size_t nw, const double* x, const double* mix,
                         double* y, char* csv, size_t csv_cap) {
    REF_TRY
    const GridSpec gi = make_grid(in_kind, in_nlat, in_nlon);
    const DiscoOperator op =
        assemble_disco(gi, make_grid(out_kind, out_nlat, out_nlon), make_basis(basis, cutoff));
    const SphericalField f = make_field(gi, cin, x);
    DistContext ctx{CommGrid(1, 1, nh, nw), {}};
    auto views = shard(ctx, std::vector<NdArray<double>>{as_tensor(f)},
                       {{1, CommAxis::polar}, {2, CommAxis::azimuth}});
    auto res = dist_disco_apply(ctx, views, op, make_mix(cout, cin, op.n_basis, mix));
    const auto glob = unshard(ctx, res, {{1, CommAxis::polar}, {2, CommAxis::azimuth}});
    std::memcpy(y, glob.data.data(), sizeof(double) * glob.data.size());
    put_csv(ctx.log, csv, csv_cap);
    REF_CATCH
}

// ---------------------------------------------------------------------------
// CPU baseline timing (bench.py --impl reference / cpu_baseline).
//
// SHT round trip with the reference's own arithmetic, on `nthreads` host threads,
// each transforming its own slice of `nfields` fields.  One-time work is hoisted
// and reported separately (the reference rebuilds tables per call,
// harmonics.hpp:159-162 / :202-205):
//   * weighted/unweighted Legendre tables are built once, rows split over threads
//     (legendre_table is per-colatitude independent, harmonics.hpp:68);
//   * the equiangular forward runs sphere::sht_forward(field, lmax, mmax, table) on a
//     field whose GridSpec is relabelled `gaussian`: harmonics.hpp:129 is a pure kind
//     check and the arithmetic below it is the one dist_sht_forward uses
//     (distsim.hpp:413-459), which is the reference's equiangular forward path.
// Returns steady-state seconds for all fields; *tables_s gets the one-time build time.
int ref_bench_sht_roundtrip(int kind, size_t nlat, size_t nlon, size_t lmax, size_t mmax,
                            size_t nfields, size_t nthreads, const double* x, double* y,
                            double* steady_s, double* tables_s) {
    REF_TRY
    using clk = std::chrono::steady_clock;
    const GridSpec g = make_grid(kind, nlat, nlon);
    if (nthreads == 0) nthreads = 1;
    auto t0 = clk::now();
    LegendreTable tw, tu;
    tw.nlat = tu.nlat = nlat;
    tw.lmax = tu.lmax = lmax;
    tw.mmax = tu.mmax = mmax;
    tw.weighted = true;
    tu.weighted = false;
    tw.values.assign(nlat * lmax * mmax, 0.0);
    tu.values.assign(nlat * lmax * mmax, 0.0);
    {
        std::vector<std::thread> th;
        const size_t per = (nlat + nthreads - 1) / nthreads;
        for (size_t t = 0; t < nthreads; ++t) {
            const size_t i0 = t * per, i1 = std::min(nlat, i0 + per);
            if (i0 >= i1) break;
            th.emplace_back([&, i0, i1] {
                std::vector<double> th_col(g.colatitudes.begin() + i0, g.colatitudes.begin() + i1);
                const LegendreTable part = legendre_table(lmax, mmax, th_col);
                const double nlon_over_dphi = static_cast<double>(g.nlon) / (2.0 * pi);
                const size_t row = lmax * mmax;
                for (size_t i = i0; i < i1; ++i) {
                    const double* src = part.values.data() + (i - i0) * row;
                    std::memcpy(tu.values.data() + i * row, src, sizeof(double) * row);
                    const double w = g.quad_weights[i] * nlon_over_dphi;  // harmonics.hpp:111
                    double* dst = tw.values.data() + i * row;
                    for (size_t k = 0; k < row; ++k) dst[k] = src[k] * w;
                }
            });
        }
        for (auto& t : th) t.join();
    }
    auto t1 = clk::now();
    GridSpec gfwd = g;
    gfwd.kind = GridKind::gaussian;
    const size_t np = nlat * nlon;
    std::vector<std::thread> th;
    std::atomic<int> err{0};
    std::string emsg;
    const size_t per = (nfields + nthreads - 1) / nthreads;
    for (size_t t = 0; t < nthreads; ++t) {
        const size_t f0 = t * per, f1 = std::min(nfields, f0 + per);
        if (f0 >= f1) break;
        th.emplace_back([&, f0, f1] {
            try {
                SphericalField f(gfwd, f1 - f0);
                std::memcpy(f.data.data(), x + f0 * np, sizeof(double) * (f1 - f0) * np);
                const SpectralCoeffs c = sht_forward(f, lmax, mmax, tw);
                const SphericalField r = sht_inverse(c, g, tu);
                if (y) std::memcpy(y + f0 * np, r.data.data(), sizeof(double) * r.data.size());
            } catch (const std::exception& e) {
                err = 1;
                emsg = e.what();
            }
        });
    }
    for (auto& t : th) t.join();
    auto t2 = clk::now();
    if (err) throw std::runtime_error(emsg);
    *tables_s = std::chrono::duration<double>(t1 - t0).count();
    *steady_s = std::chrono::duration<double>(t2 - t1).count();
    REF_CATCH
}

// DISCO apply timing with the reference's assemble_disco + disco_apply.  The c_in
// channels are split over threads: each thread applies disco_apply to its channel
// slice with the matching [c_out][c_in_slice][K] MixTensor slice (the apply is linear
// in the input channels, convolution.hpp:192-218), and the partial outputs are summed.
int ref_bench_disco(int in_kind, size_t in_nlat, size_t in_nlon, int out_kind, size_t out_nlat,
                    size_t out_nlon, int basis, double cutoff, size_t cin, size_t cout,
                    size_t nthreads, const double* x, const double* mix, double* y,
                    double* steady_s, double* assemble_s) {
    REF_TRY
    using clk = std::chrono::steady_clock;
    const GridSpec gi = make_grid(in_kind, in_nlat, in_nlon);
    const GridSpec go = make_grid(out_kind, out_nlat, out_nlon);
    auto t0 = clk::now();
    const DiscoOperator op = assemble_disco(gi, go, make_basis(basis, cutoff));
    auto t1 = clk::now();
    const size_t K = op.n_basis, npo = out_nlat * out_nlon, npi = in_nlat * in_nlon;
    if (nthreads == 0) nthreads = 1;
    const size_t per = (cin + nthreads - 1) / nthreads;
    std::vector<std::vector<double>> parts;
    std::vector<std::thread> th;
    for (size_t t = 0; t < nthreads; ++t) {
        const size_t c0 = t * per, c1 = std::min(cin, c0 + per);
        if (c0 >= c1) break;
        parts.emplace_back();
    }
    for (size_t t = 0; t < parts.size(); ++t) {
        const size_t c0 = t * per, c1 = std::min(cin, c0 + per);
        th.emplace_back([&, t, c0, c1] {
            SphericalField f(gi, c1 - c0);
            std::memcpy(f.data.data(), x + c0 * npi, sizeof(double) * f.data.size());
            MixTensor m(cout, c1 - c0, K);
            for (size_t o = 0; o < cout; ++o)
                std::memcpy(m.w.data() + o * (c1 - c0) * K, mix + (o * cin + c0) * K,
                            sizeof(double) * (c1 - c0) * K);
            parts[t] = disco_apply(op, f, m).data;
        });
    }
    for (auto& t : th) t.join();
    if (y) {
        std::memset(y, 0, sizeof(double) * cout * npo);
        for (const auto& p : parts)
            for (size_t i = 0; i < cout * npo; ++i) y[i] += p[i];
    }
    auto t2 = clk::now();
    *assemble_s = std::chrono::duration<double>(t1 - t0).count();
    *steady_s = std::chrono::duration<double>(t2 - t1).count();
    REF_CATCH
}

}  // extern "C"
