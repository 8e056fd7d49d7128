// Shared pieces of the extern "C" boundary (capi.cu, dist.cu): the opaque plan handles
// and the exception -> status-code guard (the C-ABI analogue of the reference's
// std::invalid_argument / std::runtime_error).
#pragma once

#include <new>
#include <string>

#include "disco.cuh"
#include "sht.cuh"

struct sph_sht_plan_s {
    sph::ShtPlan p;
};
struct sph_disco_plan_s {
    sph::DiscoPlan p;
};

namespace sph {
// message of the last failed call on this thread (sph_last_error)
std::string& last_error();
}  // namespace sph

namespace {
template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return SPH_OK;
    } catch (const sph::Error& e) {
        sph::last_error() = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        sph::last_error() = std::string("host allocation failed: ") + e.what();
        return SPH_ERR_OOM;
    } catch (const std::invalid_argument& e) {
        sph::last_error() = e.what();
        return SPH_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        sph::last_error() = e.what();
        return SPH_ERR_RUNTIME;
    }
}
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace
