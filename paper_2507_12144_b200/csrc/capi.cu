// extern "C" boundary of libsphgpu.so (include/sphere_gpu.h).  Converts the
// library's C++ exceptions into status codes + a thread-local message, the
// C-ABI analogue of the reference's std::invalid_argument / std::runtime_error.
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "metrics.cuh"
#include "decoder.cuh"
#include "resample.cuh"
#include "disco.cuh"
#include "sht.cuh"
#include "capi_util.cuh"

namespace sph {
std::string& last_error() {
    static thread_local std::string msg;
    return msg;
}
static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }

namespace {
struct ProfRec {
    std::string name;
    cudaEvent_t e0, e1;
    double work;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof_on{false};
std::vector<ProfRec> g_prof;
}  // namespace

ProfScope::ProfScope(const char* n, cudaStream_t s, double w) : name(n), work(w), st(s) {
    if (!g_prof_on.load(std::memory_order_relaxed)) return;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
        if (e0) cudaEventDestroy(e0);
        e0 = e1 = nullptr;
        return;
    }
    cudaEventRecord(e0, st);
}
ProfScope::~ProfScope() {
    if (!e0) return;
    cudaEventRecord(e1, st);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back(ProfRec{name, e0, e1, work});
}

cudaMemPool_t lib_pool() {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    int dev = 0;
    SPH_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(dev);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    SPH_CUDA(cudaMemPoolCreate(&pool, &props));
    uint64_t thr = ~0ull;
    SPH_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    pools[dev] = pool;
    return pool;
}
}  // namespace sph

extern "C" {

const char* sph_last_error(void) { return sph::last_error().c_str(); }
const char* sph_version(void) { return "sphgpu 0.1 sm_100a"; }
uint64_t sph_launch_count(void) { return sph::g_launches.load(); }

int sph_profile_enable(int on) {
    sph::g_prof_on.store(on != 0);
    return SPH_OK;
}

// CSV "name,launches,total_ms,work" per kernel name since the last read; resets.
int sph_profile_read(char* csv, size_t cap) {
    return guarded([&] {
        std::vector<sph::ProfRec> recs;
        {
            std::lock_guard<std::mutex> lk(sph::g_prof_mu);
            recs.swap(sph::g_prof);
        }
        std::map<std::string, std::tuple<int, double, double>> agg;
        for (auto& r : recs) {
            SPH_CUDA(cudaEventSynchronize(r.e1));
            float ms = 0.f;
            SPH_CUDA(cudaEventElapsedTime(&ms, r.e0, r.e1));
            auto& a = agg[r.name];
            std::get<0>(a) += 1;
            std::get<1>(a) += ms;
            std::get<2>(a) += r.work;
            cudaEventDestroy(r.e0);
            cudaEventDestroy(r.e1);
        }
        std::string out = "name,launches,total_ms,work\n";
        for (auto& [k, v] : agg)
            out += k + "," + std::to_string(std::get<0>(v)) + "," + std::to_string(std::get<1>(v)) +
                   "," + std::to_string(std::get<2>(v)) + "\n";
        if (csv && cap) std::snprintf(csv, cap, "%s", out.c_str());
    });
}

int sph_grid(int kind, int64_t nlat, int64_t nlon, double* colat, double* w) {
    return guarded([&] {
        std::vector<double> c, ww;
        sph::build_grid(kind, nlat, nlon, c, ww);
        std::memcpy(colat, c.data(), sizeof(double) * nlat);
        std::memcpy(w, ww.data(), sizeof(double) * nlat);
    });
}

// ------------------------------------------------------------------------ SHT
int sph_sht_plan_create(int kind, int64_t nlat, int64_t nlon, int64_t lmax, int64_t mmax,
                        int flags, sph_sht_plan* plan) {
    return guarded([&] {
        sph::require(plan != nullptr, "sph_sht_plan_create: null plan pointer");
        auto* h = new sph_sht_plan_s();
        try {
            h->p.create(kind, nlat, nlon, lmax, mmax, flags);
        } catch (...) {
            delete h;
            throw;
        }
        *plan = h;
    });
}

int sph_sht_plan_destroy(sph_sht_plan plan) {
    return guarded([&] { delete plan; });
}

int64_t sph_sht_coeffs_elems(sph_sht_plan plan, int64_t F, int layout) {
    if (!plan) return -1;
    return layout == SPH_LAYOUT_INTERNAL ? plan->p.cint_elems(F) : plan->p.dense_elems(F);
}

int64_t sph_sht_workspace_bytes(sph_sht_plan plan, int64_t F) {
    return plan ? plan->p.workspace_bytes(F) : -1;
}

int sph_sht_forward(sph_sht_plan plan, const float* x, int64_t F, float* coeffs, int layout,
                    void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "sht_forward: null plan");
        plan->p.forward(x, F, coeffs, layout, workspace, S(stream));
    });
}

int sph_sht_inverse(sph_sht_plan plan, const float* coeffs, int64_t F, int layout, float* y,
                    void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "sht_inverse: null plan");
        plan->p.inverse(coeffs, F, layout, y, workspace, S(stream));
    });
}

int sph_sht_roundtrip_host(sph_sht_plan plan, const float* xh, int64_t F, float* yh,
                           int64_t chunk) {
    return guarded([&] {
        sph::require(plan, "sht roundtrip: null plan");
        plan->p.roundtrip_host(xh, F, yh, chunk);
    });
}

int sph_sht_fft_stage(sph_sht_plan plan, const float* rings, int64_t F, int64_t h_count,
                      float* bins, void* stream) {
    return guarded([&] {
        sph::require(plan, "fft stage: null plan");
        plan->p.fft_stage(rings, F, h_count, bins, S(stream));
    });
}

int sph_sht_legendre_stage(sph_sht_plan plan, const float* bins, int64_t F, int64_t m0,
                           int64_t m_count, float* coeffs, void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "legendre stage: null plan");
        plan->p.legendre_stage(bins, F, m0, m_count, coeffs, workspace, S(stream));
    });
}

int64_t sph_sht_stage_workspace_bytes(sph_sht_plan plan, int64_t F, int64_t m_count) {
    return plan ? plan->p.stage_ws_bytes(F, m_count) : -1;
}

// ---------------------------------------------------------------------- DISCO
int sph_disco_plan_create(int in_kind, int64_t in_nlat, int64_t in_nlon, int out_kind,
                          int64_t out_nlat, int64_t out_nlon, int basis, double theta_cutoff,
                          int flags, sph_disco_plan* plan) {
    return guarded([&] {
        sph::require(plan != nullptr, "sph_disco_plan_create: null plan pointer");
        auto* h = new sph_disco_plan_s();
        try {
            h->p.create(in_kind, in_nlat, in_nlon, out_kind, out_nlat, out_nlon, basis,
                        theta_cutoff, flags);
        } catch (...) {
            delete h;
            throw;
        }
        *plan = h;
    });
}

int sph_disco_plan_destroy(sph_disco_plan plan) {
    return guarded([&] { delete plan; });
}

int sph_disco_plan_info(sph_disco_plan plan, int64_t* n_basis, int64_t* stride,
                        int64_t* nnz_per_basis) {
    return guarded([&] {
        sph::require(plan, "disco info: null plan");
        if (n_basis) *n_basis = plan->p.K;
        if (stride) *stride = plan->p.stride;
        if (nnz_per_basis) *nnz_per_basis = plan->p.nnz;
    });
}

int64_t sph_disco_workspace_bytes(sph_disco_plan plan, int64_t B, int64_t c_in, int64_t c_out) {
    return plan ? plan->p.workspace_bytes(B, c_in, c_out) : -1;
}

int sph_disco_apply(sph_disco_plan plan, const float* x, const float* mix, int64_t B,
                    int64_t c_in, int64_t c_out, float* y, void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "disco_apply: null plan");
        plan->p.apply(x, mix, B, c_in, c_out, y, workspace, S(stream));
    });
}

int64_t sph_disco_transpose_workspace_bytes(sph_disco_plan plan, int64_t B, int64_t c_in,
                                            int64_t c_out) {
    return plan ? plan->p.transpose_workspace_bytes(B, c_in, c_out) : -1;
}

int sph_disco_transpose_apply(sph_disco_plan plan, const float* v, const float* mix, int64_t B,
                              int64_t c_in, int64_t c_out, float* y, void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "disco_transpose_apply: null plan");
        plan->p.transpose_apply(v, mix, B, c_in, c_out, y, workspace, S(stream));
    });
}

int sph_disco_input_rows(sph_disco_plan plan, int64_t h_out0, int64_t n_out, int64_t* h_in0,
                         int64_t* n_in) {
    return guarded([&] {
        sph::require(plan, "disco rows: null plan");
        plan->p.input_rows(h_out0, n_out, h_in0, n_in);
    });
}

int64_t sph_disco_rows_workspace_bytes(sph_disco_plan plan, int64_t B, int64_t c_in, int64_t c_out,
                                       int64_t n_in, int64_t n_out) {
    return plan ? plan->p.rows_workspace_bytes(B, c_in, c_out, n_in, n_out) : -1;
}

int sph_disco_apply_rows(sph_disco_plan plan, const float* x, int64_t h_in0, int64_t n_in,
                         int64_t h_out0, int64_t n_out, const float* mix, int64_t B, int64_t c_in,
                         int64_t c_out, float* y, void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "disco_apply: null plan");
        plan->p.apply_rows(x, h_in0, n_in, h_out0, n_out, mix, B, c_in, c_out, y, workspace, S(stream));
    });
}

// ------------------------------------------------------------------ resample

int sph_resample_plan_create(const double* in_colat, int64_t in_nlat, int64_t in_nlon,
                             const double* out_colat, int64_t out_nlat, int64_t out_nlon,
                             sph_resample_plan* plan) {
    return guarded([&] {
        sph::require(plan && in_colat && out_colat, "bilinear_resample: null argument");
        *plan = nullptr;
        sph::ResamplePlan* p = sph::resample_new();
        try {
            sph::resample_create(*p, in_colat, in_nlat, in_nlon, out_colat, out_nlat, out_nlon);
        } catch (...) {
            sph::resample_delete(p);
            throw;
        }
        *plan = reinterpret_cast<sph_resample_plan>(p);
    });
}

int sph_resample_plan_destroy(sph_resample_plan plan) {
    return guarded([&] { sph::resample_delete(reinterpret_cast<sph::ResamplePlan*>(plan)); });
}

int64_t sph_resample_workspace_bytes(sph_resample_plan plan, int64_t C) {
    return plan ? sph::resample_workspace_bytes(*reinterpret_cast<sph::ResamplePlan*>(plan), C) : -1;
}

int sph_bilinear_resample(sph_resample_plan plan, const float* x, int64_t C, float* y, void* workspace,
                          void* stream) {
    return guarded([&] {
        sph::require(plan, "bilinear_resample: null plan");
        sph::resample_apply(*reinterpret_cast<sph::ResamplePlan*>(plan), x, C, y, workspace, S(stream));
    });
}

// ------------------------------------------------------------------ decoder
int sph_decoder_plan_create(sph_disco_plan disco, const double* latent_colat, int64_t latent_nlat,
                            int64_t latent_nlon, sph_decoder_plan* plan) {
    return guarded([&] {
        sph::require(plan && disco && latent_colat, "decode: null argument");
        *plan = nullptr;
        auto* p = new sph::DecoderPlan();
        try {
            p->create(&disco->p, latent_colat, latent_nlat, latent_nlon);
        } catch (...) {
            delete p;
            throw;
        }
        *plan = reinterpret_cast<sph_decoder_plan>(p);
    });
}

int sph_decoder_plan_destroy(sph_decoder_plan plan) {
    return guarded([&] { delete reinterpret_cast<sph::DecoderPlan*>(plan); });
}

int64_t sph_decoder_workspace_bytes(sph_decoder_plan plan, int64_t B, int64_t c_in, int64_t c_out) {
    return plan ? reinterpret_cast<sph::DecoderPlan*>(plan)->workspace_bytes(B, c_in, c_out) : -1;
}

int sph_decoder_apply(sph_decoder_plan plan, const float* latent, const float* mix, int64_t B,
                      int64_t c_in, int64_t c_out, float* y, void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "decode: null plan");
        reinterpret_cast<sph::DecoderPlan*>(plan)->apply(latent, mix, B, c_in, c_out, y, workspace, S(stream));
    });
}

int sph_weighted_crps(const float* f, const float* o, const float* w, int64_t E, int64_t C, int64_t ns,
                      int variant, double* out, void* stream) {
    return guarded([&] { sph::weighted_crps(f, o, w, E, C, ns, variant, out, S(stream)); });
}

int sph_psd_from_coeffs(const float* coeffs, int64_t F, int64_t lmax, int64_t mmax, float* psd, void* stream) {
    return guarded([&] { sph::psd_from_coeffs(coeffs, F, lmax, mmax, psd, S(stream)); });
}

int sph_spectral_crps_from_coeffs(const float* ens, const float* obs, int64_t E, int64_t C, int64_t lmax,
                                  int64_t mmax, int64_t lmax_sum, int variant, double* out, void* stream) {
    return guarded([&] {
        sph::spectral_crps_from_coeffs(ens, obs, E, C, lmax, mmax, lmax_sum, variant, out, S(stream));
    });
}

// ------------------------------------------------------ spectral conv + block
int sph_spectral_conv(sph_sht_plan plan, const float* x, const float* kernel, int64_t B,
                      int64_t c_in, int64_t c_out, int64_t klmax, float* y, void* workspace,
                      void* stream) {
    return guarded([&] {
        sph::require(plan, "spectral_conv: null plan");
        sph::spectral_conv(plan->p, x, kernel, B, c_in, c_out, klmax, y, workspace, S(stream));
    });
}

int sph_spectral_mix(sph_sht_plan plan, const float* coeffs, const float* kernel, int64_t B, int64_t c_in,
                     int64_t c_out, int64_t klmax, float* out, void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "spectral_mix: null plan");
        sph::spectral_mix(plan->p, coeffs, kernel, B, c_in, c_out, klmax, out, workspace, S(stream));
    });
}

int64_t sph_spectral_conv_workspace_bytes(sph_sht_plan plan, int64_t B, int64_t c_in,
                                          int64_t c_out) {
    return plan ? sph::spectral_conv_ws_bytes(plan->p, B, c_in, c_out) : -1;
}

int sph_block_epilogue(const float* conv, const float* x, const float* w1, const float* b1,
                       const float* w2, const float* b2, const float* scales, int64_t B, int64_t C,
                       int64_t H, int64_t npts, float* y, void* stream) {
    return guarded([&] {
        sph::block_epilogue(conv, x, w1, b1, w2, b2, scales, B, C, H, npts, y, S(stream));
    });
}

}  // extern "C"
