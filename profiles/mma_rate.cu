// Microbenchmark: sustained tcgen05.mma rate per SM on B200 (sm_100a), no data movement.
// One CTA per SM, one thread issues ITERS back-to-back MMAs into a TMEM accumulator,
// commits once, waits; reports cycles per instruction and the implied chip TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate profiles/mma_rate.cu -lcuda
// Variants: kind::tf32 / kind::f16, A from SMEM ("SS") or TMEM ("TS"), N = 64..256.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {  // K-major SWIZZLE_64B, SBO 512
    uint64_t d = (saddr >> 4) & 0x3FFF;
    d |= 1ull << 16;
    d |= static_cast<uint64_t>(512 >> 4) << 32;
    d |= 1ull << 46;
    d |= 4ull << 61;
    return d;
}
__device__ __forceinline__ uint32_t idesc(int n, bool f16) {
    uint32_t d = 1u << 4;                        // D f32
    if (f16) d |= (1u << 7) | (1u << 10);        // A/B bf16
    else d |= (2u << 7) | (2u << 10);            // A/B tf32
    d |= static_cast<uint32_t>(n >> 3) << 17;
    d |= static_cast<uint32_t>(128 >> 4) << 24;
    return d;
}

template <bool F16, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(int n, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc(n, F16);
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int k = i & 1;  // alternate the two 32-byte K halves of the 64-byte rows
            const uint64_t bd = sdesc(b0 + k * 32);
            if (TS) {
                const uint32_t ta = tm + 256 + k * 8;
                if (F16)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                                 "r"(ta), "l"(bd), "r"(id), "r"(1));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                                 "r"(ta), "l"(bd), "r"(id), "r"(1));
            } else {
                const uint64_t ad = sdesc(a0 + k * 32);
                if (F16)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                                 "l"(ad), "l"(bd), "r"(id), "r"(1));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                                 "l"(ad), "l"(bd), "r"(id), "r"(1));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar)));
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <bool F16, bool TS>
void run(int n, int sms) {
    const int iters = 4096;
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    auto k = mma_rate<F16, TS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    for (int rep = 0; rep < 2; ++rep) k<<<sms, 128, 96 * 1024>>>(n, iters, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 128, 96 * 1024>>>(n, iters, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[148];
    cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const int kk = F16 ? 16 : 8;
    const double flops = 2.0 * 128 * n * kk * iters * sms;
    printf("%-5s %s N=%3d  %7.1f cyc/mma  %7.1f TFLOP/s (event)  err=%s\n", F16 ? "f16" : "tf32",
           TS ? "TS" : "SS", n, double(mx) / iters, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    cudaFree(d);
}

// Per-iteration issue-side cost of the MMA issuer's bookkeeping (commit, waits on an
// already-completed barrier, tcgen05.fence) alone and mixed with N=192 tf32 MMAs
__global__ void __launch_bounds__(128, 1) issue_cost(int mode, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar[2];
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc(192, false);
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
        const uint32_t b = smem_u32(&bar[0]), done = smem_u32(&bar[1]);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b));  // phase 0 complete
        const long long t0 = clock64();
        auto mmas = [&](int nm) {
            for (int m = 0; m < nm; ++m)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                             "l"(sdesc(a0 + (m & 1) * 32)), "l"(sdesc(b0 + (m & 1) * 32)), "r"(id), "r"(1));
        };
        auto wait_done = [&]() {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok)
                             : "r"(b));
        };
        auto test_done = [&]() {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok)
                             : "r"(b));
        };
        auto fence = [&]() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); };
        auto commit = [&]() {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(done));
        };
        for (int i = 0; i < iters; ++i) {
            switch (mode) {
                case 0: commit(); break;
                case 1: wait_done(); break;
                case 2: fence(); break;
                case 3: test_done(); break;
                case 4: mmas(6); commit(); break;
                case 5: mmas(12); commit(); break;
                case 6: wait_done(); fence(); mmas(6); commit(); break;             // old loop
                case 7: wait_done(); fence(); mmas(4); wait_done(); fence(); mmas(2); commit(); break;  // ALO lag
                case 8: wait_done(); fence(); mmas(12); commit(); break;            // BK=32
                case 9: test_done(); fence(); mmas(6); commit(); break;
                case 10: wait_done(); mmas(6); commit(); break;                      // no fence
                case 11: mmas(6); break;
            }
        }
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        long long* d;
        cudaMalloc(&d, sms * sizeof(long long));
        cudaFuncSetAttribute(issue_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        const char* names[] = {"commit", "try_wait(done)", "fence::after", "test_wait(done)", "6 mma + commit",
                               "12 mma + commit", "wait+fence+6mma+commit", "2x(wait+fence)+4+2mma+commit",
                               "wait+fence+12mma+commit", "test+fence+6mma+commit", "wait+6mma+commit", "6 mma"};
        for (int mode = 0; mode < 12; ++mode) {
            if (only >= 0 && mode != only) continue;
            const int iters = 2048;
            issue_cost<<<sms, 128, 64 * 1024>>>(mode, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148], mx = 0;
            cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
            for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("%-22s %8.1f cyc/iter (issue side)  %s\n", names[mode], double(mx) / iters, cudaGetErrorString(e));
        }
        cudaFree(d);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int n : {64, 128, 192, 256}) {
        run<false, false>(n, sms);
        run<false, true>(n, sms);
        run<true, false>(n, sms);
        run<true, true>(n, sms);
    }
    return 0;
}
