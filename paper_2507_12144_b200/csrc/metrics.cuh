// SHT-consumer reductions (metrics.hpp:300-314, loss.hpp:37-81), implemented in metrics.cu.
#pragma once

#include "common.cuh"

namespace sph {
void psd_from_coeffs(const float* coeffs, int64_t F, int64_t lmax, int64_t mmax, float* psd, cudaStream_t st);
void spectral_crps_from_coeffs(const float* ens, const float* obs, int64_t E, int64_t C, int64_t lmax,
                               int64_t mmax, int64_t lmax_sum, int variant, double* out, cudaStream_t st);
void weighted_crps(const float* f, const float* o, const float* w, int64_t E, int64_t C, int64_t ns, int variant,
                   double* out, cudaStream_t st);
}  // namespace sph
