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

// Makes `dev` current for the scope and restores the caller's device afterwards (plans
// are bound to the device they were created on; the caller's current device is theirs).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        SPH_CUDA(cudaGetDevice(&prev));
        if (prev != dev) SPH_CUDA(cudaSetDevice(dev));
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Rejects a device pointer that lives on a device other than the plan's (a tensor on
// cuda:1 handed to a cuda:0 plan).  Host / unregistered pointers pass: they are the
// caller's business (and fail loudly in the kernel if wrong).
inline void require_on_device(const void* ptr, int dev, const char* what) {
    if (!ptr) return;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    if (a.type == cudaMemoryTypeDevice && a.device != dev)
        fail(SPH_ERR_INVALID_ARGUMENT, std::string(what) + ": buffer is on cuda:" + std::to_string(a.device) +
                                           ", the plan on cuda:" + std::to_string(dev));
}

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

// Library-owned stream-ordered memory pool of the current device (created once, release
// threshold UINT64_MAX so transient workspaces stay mapped between calls) and an RAII
// allocation from it that is freed stream-ordered on scope exit, including unwinding.
cudaMemPool_t lib_pool();
struct StreamBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    StreamBuf(size_t bytes, cudaStream_t s) : st(s) {
        if (bytes) SPH_CUDA(cudaMallocFromPoolAsync(&p, bytes, lib_pool(), st));
    }
    ~StreamBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    StreamBuf(const StreamBuf&) = delete;
    StreamBuf& operator=(const StreamBuf&) = delete;
};

// Kernel-launch counter: every kernel launched by the library bumps it (bench.py
// reports it as gpu_launches).
void count_launch(int n = 1);

// Stream-ordered per-kernel timing (sph_profile_enable / sph_profile_read): when
// enabled, a ProfScope records a CUDA event pair on the launching stream around the
// launch it wraps; durations are summed per name when read.  The scope owns its events
// and hands the finished record to the profile list in its destructor, so a concurrent
// sph_profile_read never sees (or invalidates) a record that is still open.
struct ProfScope {
    ProfScope(const char* name, cudaStream_t st, double work = 0.0);
    ~ProfScope();
    const char* name = nullptr;
    double work = 0.0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaStream_t st;
};

}  // namespace sph
