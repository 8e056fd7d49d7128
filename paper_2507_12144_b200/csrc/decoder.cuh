// Fused decoder (model.hpp:372-394 decode_preclamp, one channel group):
// y = disco_apply(dec_op, bilinear_resample(latent, out_grid), mix).
#pragma once

#include "disco.cuh"
#include "resample.cuh"

namespace sph {

struct DecoderPlan {
    DiscoPlan* disco = nullptr;  // borrowed: the out_grid -> out_grid operator (dec_op)
    ResamplePlan rs;             // latent grid -> disco's input grid
    FftPlan fft_lat;             // latent ring length
    bool fourier = false;        // integer longitude ratio and a Fourier-path DISCO
    int ratio = 0;
    int64_t nbl = 0;             // latent half-spectrum bins
    DevBuf<float> d_h;           // Fejer response of the longitude hat interpolant per bin
    std::mutex mu;
    DevBuf<uint8_t> own_ws;

    void create(DiscoPlan* d, const double* lat_colat, int64_t lat_nlat, int64_t lat_nlon);
    int64_t workspace_bytes(int64_t B, int64_t cin, int64_t cout) const;
    void apply(const float* latent, const float* mix, int64_t B, int64_t cin, int64_t cout, float* y,
               void* ws, cudaStream_t st);
};

}  // namespace sph
