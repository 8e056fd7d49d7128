// Shared helpers for the sm_100a spherical-operator library (libsphgpu.so).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/sphere_gpu.h"

namespace sph {

// Error classes mirror the reference's exceptions: invalid_argument ->
// SPH_ERR_INVALID_ARGUMENT, runtime_error -> SPH_ERR_RUNTIME; CUDA/NCCL/OOM get
// their own codes.  Thrown inside the library, converted to status codes at the
// C-ABI boundary (capi.cu).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const std::string& msg) {
    if (!ok) fail(SPH_ERR_INVALID_ARGUMENT, msg);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        fail(e == cudaErrorMemoryAllocation ? SPH_ERR_OOM : SPH_ERR_CUDA,
             std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                 std::to_string(line) + ")");
    }
}
#define SPH_CUDA(x) ::sph::cuda_check((x), #x, __FILE__, __LINE__)
#define SPH_LAUNCH_CHECK() ::sph::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

inline int num_sms() {
    static int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return n;
}

inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Device buffer owned by a plan (RAII).
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count, bool zero = true) { alloc(count, zero); }
    void alloc(size_t count, bool zero = true) {
        release();
        n = count;
        if (count) {
            SPH_CUDA(cudaMalloc(&p, count * sizeof(T)));
            if (zero) SPH_CUDA(cudaMemset(p, 0, count * sizeof(T)));
        }
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// Kernel-launch counter: every kernel launched by the library bumps it (bench.py
// reports it as gpu_launches).
void count_launch(int n = 1);

// Stream-ordered per-kernel timing (sph_profile_enable / sph_profile_read): when
// enabled, a ProfScope records a CUDA event pair on the launching stream around the
// launch it wraps; durations are summed per name when read.
struct ProfScope {
    ProfScope(const char* name, cudaStream_t st, double work = 0.0);
    ~ProfScope();
    int slot = -1;
    cudaStream_t st;
};

}  // namespace sph
