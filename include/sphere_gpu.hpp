// sphere_gpu.hpp -- C++ drop-in shim over the C ABI (sphere_gpu.h) for callers of the
// reference library spheretk.  Same value semantics, signatures and exception types as
// namespace sphere (/root/reference/proj/include/sphere/):
//
//   sphere::sht_forward(field, lmax, mmax)        -> sphere_gpu::sht_forward(...)
//   sphere::sht_inverse(coeffs, grid)             -> sphere_gpu::sht_inverse(...)
//   sphere::disco_apply(op, field, mix)           -> sphere_gpu::disco_apply(op, field, mix)
//   sphere::disco_transpose_apply(op, field, mix) -> sphere_gpu::disco_transpose_apply(...)
//       with op = sphere_gpu::assemble_disco(in_grid, out_grid, basis)
//   sphere::spectral_conv(field, kernel)          -> sphere_gpu::spectral_conv(...)
//
// fp64 host data are converted to fp32 device buffers, the work runs in libsphgpu.so
// (sm_100a), results come back as fp64 reference types.  Plans are cached per
// (grid, lmax, mmax) / (grids, basis), replacing the per-call table builds of
// harmonics.hpp:159-162 / :202-205.  Status codes map back to the reference's
// exceptions: SPH_ERR_INVALID_ARGUMENT -> std::invalid_argument, everything else ->
// std::runtime_error.  Include after the reference headers; link -lsphgpu -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "sphere/convolution.hpp"
#include "sphere/field.hpp"
#include "sphere/harmonics.hpp"
#include "sphere_gpu.h"

namespace sphere_gpu {

inline void check(int rc) {
    if (rc == SPH_OK) return;
    const std::string msg = sph_last_error();
    if (rc == SPH_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

namespace detail {

template <class T>
struct DeviceArray {
    T* p = nullptr;
    size_t n = 0;
    explicit DeviceArray(size_t count) : n(count) {
        if (count && cudaMalloc(&p, count * sizeof(T)) != cudaSuccess)
            throw std::runtime_error("sphere_gpu: device allocation failed");
    }
    ~DeviceArray() {
        if (p) cudaFree(p);
    }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    void upload(const std::vector<float>& h) {
        if (cudaMemcpy(p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
            throw std::runtime_error("sphere_gpu: H2D copy failed");
    }
    std::vector<float> download() const {
        std::vector<float> h(n);
        if (cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess)
            throw std::runtime_error("sphere_gpu: D2H copy failed");
        return h;
    }
};

inline int kind_of(const sphere::GridSpec& g) {
    return g.kind == sphere::GridKind::equiangular ? SPH_EQUIANGULAR : SPH_GAUSSIAN;
}

inline std::vector<float> to_f32(const std::vector<double>& v) {
    return std::vector<float>(v.begin(), v.end());
}

struct ShtPlanHandle {
    sph_sht_plan h = nullptr;
    ~ShtPlanHandle() {
        if (h) sph_sht_plan_destroy(h);
    }
};

inline sph_sht_plan sht_plan(const sphere::GridSpec& g, size_t lmax, size_t mmax, int flags) {
    static std::mutex mu;
    static std::map<std::tuple<int, size_t, size_t, size_t, size_t, int>, std::unique_ptr<ShtPlanHandle>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = cache[std::make_tuple(kind_of(g), g.nlat, g.nlon, lmax, mmax, flags)];
    if (!slot) {
        auto h = std::make_unique<ShtPlanHandle>();
        check(sph_sht_plan_create(kind_of(g), static_cast<int64_t>(g.nlat), static_cast<int64_t>(g.nlon),
                                  static_cast<int64_t>(lmax), static_cast<int64_t>(mmax), flags, &h->h));
        slot = std::move(h);
    }
    return slot->h;
}

inline sphere::SpectralCoeffs forward_impl(const sphere::SphericalField& field, size_t lmax,
                                           size_t mmax, int flags) {
    sphere::require_same_sampling(field, field.grid, "sht_forward");
    sph_sht_plan p = sht_plan(field.grid, lmax, mmax, flags);
    const size_t F = field.channels, np = field.npoints();
    DeviceArray<float> x(F * np), c(F * lmax * mmax * 2);
    x.upload(to_f32(field.data));
    check(sph_sht_forward(p, x.p, static_cast<int64_t>(F), c.p, SPH_LAYOUT_DENSE_LM, nullptr, nullptr));
    const std::vector<float> h = c.download();
    sphere::SpectralCoeffs out(lmax, mmax, F);
    for (size_t i = 0; i < out.coeffs.size(); ++i) out.coeffs[i] = {h[2 * i], h[2 * i + 1]};
    return out;
}

}  // namespace detail

// harmonics.hpp:126-169 (Gaussian grids only, exactly like the reference)
inline sphere::SpectralCoeffs sht_forward(const sphere::SphericalField& field, size_t lmax,
                                          size_t mmax) {
    const sphere::GridSpec& g = field.grid;
    if (g.kind != sphere::GridKind::gaussian)
        throw std::invalid_argument("sht_forward: requires a gaussian grid");
    if (g.nlat < lmax || g.nlon < 2 * mmax)
        throw std::invalid_argument("sht_forward: resolution insufficient for lmax/mmax");
    return detail::forward_impl(field, lmax, mmax, SPH_PREC_3XTF32);
}

inline sphere::SpectralCoeffs sht_forward(const sphere::SphericalField& field) {
    const size_t lmax = field.grid.nlat;
    const size_t mmax = std::min(sphere::default_mmax(lmax, field.grid.nlon), field.grid.nlon / 2);
    return sphere_gpu::sht_forward(field, lmax, std::max<size_t>(mmax, 1));
}

// The reference's equiangular forward (dist_sht_forward on a 1x1 CommGrid,
// distsim.hpp:404-463) as a plain call: any grid kind.
inline sphere::SpectralCoeffs sht_forward_any_grid(const sphere::SphericalField& field,
                                                   size_t lmax, size_t mmax) {
    return detail::forward_impl(field, lmax, mmax,
                                SPH_PREC_3XTF32 | SPH_FLAG_ALLOW_EQUIANGULAR_FORWARD);
}

// harmonics.hpp:173-205
inline sphere::SphericalField sht_inverse(const sphere::SpectralCoeffs& coeffs,
                                          const sphere::GridSpec& grid) {
    sph_sht_plan p = detail::sht_plan(grid, coeffs.lmax, coeffs.mmax, SPH_PREC_3XTF32);
    const size_t F = coeffs.channels, np = grid.nlat * grid.nlon;
    std::vector<float> hc(coeffs.coeffs.size() * 2);
    for (size_t i = 0; i < coeffs.coeffs.size(); ++i) {
        hc[2 * i] = static_cast<float>(coeffs.coeffs[i].real());
        hc[2 * i + 1] = static_cast<float>(coeffs.coeffs[i].imag());
    }
    detail::DeviceArray<float> c(hc.size()), y(F * np);
    c.upload(hc);
    check(sph_sht_inverse(p, c.p, static_cast<int64_t>(F), SPH_LAYOUT_DENSE_LM, y.p, nullptr, nullptr));
    const std::vector<float> h = y.download();
    sphere::SphericalField out(grid, F);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = h[i];
    return out;
}

// convolution.hpp:141-177: the assembled operator lives on the device
struct DiscoOperator {
    sphere::GridSpec in_grid, out_grid;
    size_t n_basis = 0, stride = 1;
    std::shared_ptr<sph_disco_plan_s> plan;
};

inline DiscoOperator assemble_disco(const sphere::GridSpec& in_grid, const sphere::GridSpec& out_grid,
                                    const sphere::FilterBasis& basis) {
    const bool iso = basis.indices.size() == 1 && basis.indices[0] == std::make_pair(0, 0);
    const bool morlet = basis.indices == sphere::morlet_basis(basis.theta_cutoff).indices;
    if (!iso && !morlet) throw std::invalid_argument("assemble_disco: only the Morlet and isotropic bases");
    sph_disco_plan h = nullptr;
    check(sph_disco_plan_create(detail::kind_of(in_grid), static_cast<int64_t>(in_grid.nlat),
                                static_cast<int64_t>(in_grid.nlon), detail::kind_of(out_grid),
                                static_cast<int64_t>(out_grid.nlat), static_cast<int64_t>(out_grid.nlon),
                                iso ? SPH_BASIS_ISOTROPIC : SPH_BASIS_MORLET, basis.theta_cutoff,
                                SPH_PREC_3XTF32, &h));
    DiscoOperator op;
    op.in_grid = in_grid;
    op.out_grid = out_grid;
    op.plan = std::shared_ptr<sph_disco_plan_s>(h, [](sph_disco_plan p) { sph_disco_plan_destroy(p); });
    int64_t k = 0, s = 0, nnz = 0;
    check(sph_disco_plan_info(h, &k, &s, &nnz));
    op.n_basis = static_cast<size_t>(k);
    op.stride = static_cast<size_t>(s);
    return op;
}

// convolution.hpp:181-220
inline sphere::SphericalField disco_apply(const DiscoOperator& op, const sphere::SphericalField& field,
                                          const sphere::MixTensor& mix) {
    sphere::require_same_sampling(field, op.in_grid, "disco_apply");
    if (mix.c_in != field.channels || mix.k != op.n_basis)
        throw std::invalid_argument("disco_apply: mix tensor shape mismatch");
    detail::DeviceArray<float> x(field.data.size()), w(mix.w.size()),
        y(mix.c_out * op.out_grid.nlat * op.out_grid.nlon);
    x.upload(detail::to_f32(field.data));
    w.upload(detail::to_f32(mix.w));
    check(sph_disco_apply(op.plan.get(), x.p, w.p, 1, static_cast<int64_t>(mix.c_in),
                          static_cast<int64_t>(mix.c_out), y.p, nullptr, nullptr));
    const std::vector<float> h = y.download();
    sphere::SphericalField out(op.out_grid, mix.c_out);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = h[i];
    return out;
}

// convolution.hpp:226-266 (field on the output grid -> result on the input grid)
inline sphere::SphericalField disco_transpose_apply(const DiscoOperator& op,
                                                    const sphere::SphericalField& field,
                                                    const sphere::MixTensor& mix) {
    sphere::require_same_sampling(field, op.out_grid, "disco_transpose_apply");
    if (mix.c_in == 0 || mix.k != op.n_basis)
        throw std::invalid_argument("disco_transpose_apply: mix tensor shape mismatch");
    if (mix.c_out != field.channels)
        throw std::invalid_argument("disco_transpose_apply: mix tensor shape mismatch");
    detail::DeviceArray<float> v(field.data.size()), w(mix.w.size()),
        y(mix.c_in * op.in_grid.nlat * op.in_grid.nlon);
    v.upload(detail::to_f32(field.data));
    w.upload(detail::to_f32(mix.w));
    check(sph_disco_transpose_apply(op.plan.get(), v.p, w.p, 1, static_cast<int64_t>(mix.c_in),
                                    static_cast<int64_t>(mix.c_out), y.p, nullptr, nullptr));
    const std::vector<float> h = y.download();
    sphere::SphericalField out(op.in_grid, mix.c_in);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = h[i];
    return out;
}

// convolution.hpp:286-304
inline sphere::SphericalField spectral_conv(const sphere::SphericalField& field,
                                            const sphere::SpectralKernel& kernel) {
    if (field.grid.kind != sphere::GridKind::gaussian)
        throw std::invalid_argument("spectral_conv: requires a gaussian grid");
    if (kernel.c_in != field.channels) throw std::invalid_argument("spectral_conv: kernel channel mismatch");
    const size_t lmax = std::min(kernel.lmax, field.grid.nlat);
    const size_t mmax = std::min(lmax, field.grid.nlon / 2);
    sph_sht_plan p = detail::sht_plan(field.grid, lmax, mmax, SPH_PREC_3XTF32);
    const size_t np = field.npoints();
    detail::DeviceArray<float> x(field.data.size()), k(kernel.k.size()), y(kernel.c_out * np);
    x.upload(detail::to_f32(field.data));
    k.upload(detail::to_f32(kernel.k));
    const int64_t ws = sph_spectral_conv_workspace_bytes(p, 1, static_cast<int64_t>(kernel.c_in),
                                                         static_cast<int64_t>(kernel.c_out));
    detail::DeviceArray<unsigned char> w(static_cast<size_t>(ws));
    check(sph_spectral_conv(p, x.p, k.p, 1, static_cast<int64_t>(kernel.c_in),
                            static_cast<int64_t>(kernel.c_out), static_cast<int64_t>(kernel.lmax), y.p,
                            w.p, nullptr));
    const std::vector<float> h = y.download();
    sphere::SphericalField out(field.grid, kernel.c_out);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = h[i];
    return out;
}

}  // namespace sphere_gpu
