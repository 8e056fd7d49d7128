// bilinear_resample plan (resample.hpp:20-114), implemented in resample.cu.
#pragma once

#include <vector>

#include "common.cuh"

namespace sph {
// bracketing tables (host fp64 -> device): output row oi interpolates the pole-extended
// input rows i0[oi], i1[oi] with weight wt[oi] on i1; extended row 0 is the north pole
// (ring mean of input row 0) when add_north, row ext_nlat-1 the south pole when add_south
struct ResamplePlan {
    int device = 0;
    int64_t in_nlat = 0, in_nlon = 0, out_nlat = 0, out_nlon = 0;
    bool ext = false, add_north = false, add_south = false;
    int64_t ext_nlat = 0;
    std::vector<int32_t> i0, i1, j0, j1;
    std::vector<double> wt, wp;
    DevBuf<int32_t> d_i0, d_i1, d_j0, d_j1;
    DevBuf<float> d_wt, d_wp;
};
ResamplePlan* resample_new();
void resample_delete(ResamplePlan* p);
void resample_create(ResamplePlan& p, const double* in_colat, int64_t in_nlat, int64_t in_nlon,
                     const double* out_colat, int64_t out_nlat, int64_t out_nlon);
int64_t resample_workspace_bytes(const ResamplePlan& p, int64_t C);
void resample_apply(const ResamplePlan& p, const float* x, int64_t C, float* y, void* ws, cudaStream_t st);
}  // namespace sph
