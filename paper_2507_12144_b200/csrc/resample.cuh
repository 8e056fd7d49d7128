// bilinear_resample plan (resample.hpp:20-114), implemented in resample.cu.
#pragma once

#include "common.cuh"

namespace sph {
struct ResamplePlan;
ResamplePlan* resample_new();
void resample_delete(ResamplePlan* p);
void resample_create(ResamplePlan& p, const double* in_colat, int64_t in_nlat, int64_t in_nlon,
                     const double* out_colat, int64_t out_nlat, int64_t out_nlon);
int64_t resample_workspace_bytes(const ResamplePlan& p, int64_t C);
void resample_apply(const ResamplePlan& p, const float* x, int64_t C, float* y, void* ws, cudaStream_t st);
}  // namespace sph
