// Microbenchmark: TMA load throughput per SM on B200 (sm_100a).
// One CTA per SM; one thread keeps S stages in flight, each stage one load into SMEM,
// waits stage full barriers round-robin and re-issues.  Reports aggregate GB/s.
//   mode 0: 2D tensor box {32 fp32 (128 B, SWIZZLE_128B), ROWS rows} from a row-major
//           [rows x 384] fp32 matrix, walking k-blocks of 128-row tiles (the GEMM's A loads)
//   mode 1: 1D cp.async.bulk of ROWS*128 contiguous bytes (same bytes per load)
//   footprint: "l2" = 32 MB source (L2 resident after warm-up), "hbm" = 4 GB source
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate profiles/tma_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void __launch_bounds__(32, 1)
tma_rate(const __grid_constant__ CUtensorMap map, const float* src, int64_t src_rows, int rows_box,
         int stages, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[16];
    const uint32_t stage_bytes = rows_box * 128;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const int64_t tiles = src_rows / 128;
    // each CTA walks its own sequence of (tile, k-block): tile = (cta + i / 12 * grid) % tiles
    auto issue = [&](int i, int s) {
        const int64_t tile = (blockIdx.x + static_cast<int64_t>(i / 12) * gridDim.x) % tiles;
        const int kb = i % 12;
        const uint32_t b = smem_u32(&bar[s]);
        const uint32_t dst = smem_u32(sm) + s * stage_bytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(stage_bytes));
        if (MODE == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(kb * 32), "r"(static_cast<int>(tile * 128)), "r"(b)
                : "memory");
        } else {
            const int64_t chunks = src_rows * 384 * 4 / stage_bytes;
            const char* g = reinterpret_cast<const char*>(src) + ((tile * 12 + kb) % chunks) * static_cast<int64_t>(stage_bytes);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "l"(g), "r"(stage_bytes), "r"(b)
                : "memory");
        }
    };
    for (int s = 0; s < stages; ++s) issue(s, s);
    const long long t0 = clock64();
    int s = 0;
    uint32_t ph = 0;
    for (int i = stages; i < iters + stages; ++i) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar[s])), "r"(ph));
        if (i < iters) issue(i, s);
        if (++s == stages) { s = 0; ph ^= 1; }
    }
    out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
    const int64_t cols = 384;  // 12 k-blocks of 32
    long long* d_out;
    cudaMalloc(&d_out, sms * sizeof(long long));
    for (int big = 0; big < 2; ++big) {
        const int64_t bytes = big ? (4LL << 30) : (32LL << 20);
        const int64_t rows = bytes / (cols * 4) / 128 * 128;
        float* src;
        if (cudaMalloc(&src, rows * cols * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
        cudaMemset(src, 0, rows * cols * 4);
        for (int rows_box : {128, 256}) {
            CUtensorMap map;
            cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
            cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 4)};
            cuuint32_t box[2] = {32, static_cast<cuuint32_t>(rows_box)};
            cuuint32_t es[2] = {1, 1};
            enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            for (int mode = 0; mode < 2; ++mode)
                for (int stages : {2, 4, 8}) {
                    const int smem = stages * rows_box * 128;
                    if (smem > 200 * 1024) continue;
                    const int iters = big ? 2000 : 4000;
                    auto k = mode == 0 ? tma_rate<0> : tma_rate<1>;
                    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                    k<<<sms, 32, smem>>>(map, src, rows, rows_box, stages, iters, d_out);
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0);
                    cudaEventCreate(&e1);
                    cudaEventRecord(e0);
                    k<<<sms, 32, smem>>>(map, src, rows, rows_box, stages, iters, d_out);
                    cudaEventRecord(e1);
                    cudaError_t err = cudaDeviceSynchronize();
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    const double gbs = double(iters) * rows_box * 128 * sms / (ms * 1e-3) / 1e9;
                    printf("%-4s %-6s box %3d rows  stages %d  in-flight %3d KB/SM  %7.0f GB/s  %s\n",
                           big ? "hbm" : "l2", mode == 0 ? "tensor" : "bulk1d", rows_box, stages,
                           smem / 1024, gbs, cudaGetErrorString(err));
                }
        }
        cudaFree(src);
    }
    return 0;
}
