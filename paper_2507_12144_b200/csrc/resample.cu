// bilinear_resample with pole extension (resample.hpp:20-114) on sm_100a.
//
// The plan computes, on the host in fp64 and in the reference's exact order of
// operations, the bracketing latitude rows (upper_bound over the pole-extended
// colatitudes, ties resolved to weight 0 for the upper row) and longitude columns
// (position snapping within 1e-12, modular wrap) of every output row / column.  The
// device work is two memory-bound passes: per-field pole means of the first / last input
// ring (only when the output reaches beyond the input's latitudes, :70-74), then one
// four-term gather per output sample (thread per sample, consecutive threads ->
// consecutive output longitudes; the two input rows of an output row stay in L1/L2).
#include <algorithm>
#include <cmath>
#include <vector>

#include "resample.cuh"

namespace sph {


namespace {
constexpr double kPi = 3.14159265358979323846;

// mean of ring 0 (north, slot 0) and ring nlat-1 (south, slot 1) of each field
__global__ void pole_mean_kernel(const float* __restrict__ x, int64_t nlat, int64_t nlon,
                                 float* __restrict__ means) {
    const int64_t c = blockIdx.x;
    const int which = blockIdx.y;
    const float* row = x + (c * nlat + (which ? nlat - 1 : 0)) * nlon;
    float s = 0.f;
    for (int64_t j = threadIdx.x; j < nlon; j += blockDim.x) s += row[j];
    __shared__ float red[32];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) means[c * 2 + which] = s / static_cast<float>(nlon);
    }
}

__global__ void bilinear_kernel(const float* __restrict__ x, int64_t in_nlat, int64_t in_nlon,
                                int64_t out_nlat, int64_t out_nlon, int row0, int north_row, int south_row,
                                const int32_t* __restrict__ i0s, const int32_t* __restrict__ i1s,
                                const float* __restrict__ wts, const int32_t* __restrict__ j0s,
                                const int32_t* __restrict__ j1s, const float* __restrict__ wps,
                                const float* __restrict__ means, float* __restrict__ y) {
    const int64_t oj = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t oi = blockIdx.y, c = blockIdx.z;
    if (oj >= out_nlon) return;
    const int i0 = i0s[oi], i1 = i1s[oi];
    const float wt = wts[oi];
    const int j0 = j0s[oj], j1 = j1s[oj];
    const float wp = wps[oj];
    const float* xc = x + c * in_nlat * in_nlon;
    // extended-grid row -> value at column j (pole rows are the ring means)
    auto v = [&](int er, int j) -> float {
        if (er == north_row) return means[c * 2];
        if (er == south_row) return means[c * 2 + 1];
        return __ldg(xc + static_cast<int64_t>(er - row0) * in_nlon + j);
    };
    y[(c * out_nlat + oi) * out_nlon + oj] = (1.f - wt) * (1.f - wp) * v(i0, j0) + wt * (1.f - wp) * v(i1, j0) +
                                             (1.f - wt) * wp * v(i0, j1) + wt * wp * v(i1, j1);
}

template <class T>
void upload(DevBuf<T>& d, const std::vector<T>& h) {
    d.alloc(std::max<size_t>(h.size(), 1), false);
    if (!h.empty()) SPH_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}
}  // namespace

void resample_create(ResamplePlan& p, const double* in_colat, int64_t in_nlat, int64_t in_nlon,
                     const double* out_colat, int64_t out_nlat, int64_t out_nlon) {
    require(in_nlat >= 1 && in_nlon >= 1 && out_nlat >= 1 && out_nlon >= 1, "bilinear_resample: empty grid");
    require(in_nlat < (1LL << 30) && out_nlat <= 65535, "bilinear_resample: grid too large");
    SPH_CUDA(cudaGetDevice(&p.device));
    p.in_nlat = in_nlat;
    p.in_nlon = in_nlon;
    p.out_nlat = out_nlat;
    p.out_nlon = out_nlon;
    // resample.hpp:68-73: extend to the poles only when the output leaves the input's range
    p.ext = out_colat[0] < in_colat[0] || out_colat[out_nlat - 1] > in_colat[in_nlat - 1];
    p.add_north = p.ext && in_colat[0] > 0.0;
    p.add_south = p.ext && in_colat[in_nlat - 1] < kPi;
    std::vector<double> ec;
    if (p.add_north) ec.push_back(0.0);
    ec.insert(ec.end(), in_colat, in_colat + in_nlat);
    if (p.add_south) ec.push_back(kPi);
    p.ext_nlat = static_cast<int64_t>(ec.size());
    const int64_t n = p.ext_nlat;
    std::vector<int32_t>&i0 = p.i0, &i1 = p.i1, &j0 = p.j0, &j1 = p.j1;
    std::vector<double>&wt = p.wt, &wp = p.wp;
    i0.assign(out_nlat, 0);
    i1.assign(out_nlat, 0);
    j0.assign(out_nlon, 0);
    j1.assign(out_nlon, 0);
    wt.assign(out_nlat, 0.0);
    wp.assign(out_nlon, 0.0);
    for (int64_t oi = 0; oi < out_nlat; ++oi) {  // :81-90
        const double theta = out_colat[oi];
        const int64_t u = std::upper_bound(ec.begin(), ec.end(), theta) - ec.begin();
        int64_t a1 = u, a0 = u > 0 ? u - 1 : 0;
        if (a1 >= n) a1 = n - 1;
        const double t0 = ec[a0], t1 = ec[a1];
        const double w = (a1 == a0 || theta <= t0) ? 0.0 : (theta - t0) / (t1 - t0);
        i0[oi] = static_cast<int32_t>(a0);
        i1[oi] = static_cast<int32_t>(a1);
        wt[oi] = w;
    }
    const double dphi = 2.0 * kPi / static_cast<double>(in_nlon);
    for (int64_t oj = 0; oj < out_nlon; ++oj) {  // :92-105
        const double phi = 2.0 * kPi * static_cast<double>(oj) / static_cast<double>(out_nlon);
        const double pos = phi / dphi;
        int64_t a0 = std::min<int64_t>(static_cast<int64_t>(pos), in_nlon - 1);
        double w = pos - static_cast<double>(a0);
        if (w < 1e-12) {
            w = 0.0;
        } else if (w > 1.0 - 1e-12) {
            a0 = (a0 + 1) % in_nlon;
            w = 0.0;
        }
        j0[oj] = static_cast<int32_t>(a0);
        j1[oj] = static_cast<int32_t>((a0 + 1) % in_nlon);
        wp[oj] = w;
    }
    upload(p.d_i0, i0);
    upload(p.d_i1, i1);
    upload(p.d_wt, std::vector<float>(wt.begin(), wt.end()));
    upload(p.d_j0, j0);
    upload(p.d_j1, j1);
    upload(p.d_wp, std::vector<float>(wp.begin(), wp.end()));
}

ResamplePlan* resample_new() { return new ResamplePlan(); }
void resample_delete(ResamplePlan* p) { delete p; }

int64_t resample_workspace_bytes(const ResamplePlan& p, int64_t C) {
    return (p.add_north || p.add_south) ? C * 2 * 4 + 256 : 256;
}

void resample_apply(const ResamplePlan& p, const float* x, int64_t C, float* y, void* ws, cudaStream_t st) {
    require(C >= 0, "bilinear_resample: negative field count");
    require(C <= 65535, "bilinear_resample: at most 65535 fields per call");
    if (C == 0) return;
    DeviceGuard dguard(p.device);
    float* means = static_cast<float*>(ws);
    if (p.add_north || p.add_south) {
        require(means != nullptr, "bilinear_resample: workspace required for the pole extension");
        pole_mean_kernel<<<dim3(static_cast<unsigned>(C), 2), 256, 0, st>>>(x, p.in_nlat, p.in_nlon, means);
        SPH_LAUNCH_CHECK();
        count_launch();
    }
    const int row0 = p.add_north ? 1 : 0;
    const int north = p.add_north ? 0 : -1, south = p.add_south ? static_cast<int>(p.ext_nlat - 1) : -1;
    dim3 grid(static_cast<unsigned>((p.out_nlon + 255) / 256), static_cast<unsigned>(p.out_nlat),
              static_cast<unsigned>(C));
    {
        ProfScope prof("bilinear_resample", st, 4.0 * C * (p.in_nlat * p.in_nlon + p.out_nlat * p.out_nlon));
        bilinear_kernel<<<grid, 256, 0, st>>>(x, p.in_nlat, p.in_nlon, p.out_nlat, p.out_nlon, row0, north, south,
                                              p.d_i0.p, p.d_i1.p, p.d_wt.p, p.d_j0.p, p.d_j1.p, p.d_wp.p, means, y);
        SPH_LAUNCH_CHECK();
    }
    count_launch();
}

}  // namespace sph
