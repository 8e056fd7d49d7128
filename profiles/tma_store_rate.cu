// Microbenchmark: TMA tensor STORE rate (SMEM -> HBM) by inner box width (B200).
// The inverse Legendre GEMM's epilogue stores 32 x 32 fp32 chunks of the EOi operand as
// box {32, 1, 1, 32} of a [n][t][g][128] map: 128-byte inner runs, 4 KB per store.
//   mode 0: box {32, 32} over a [rows][128] fp32 matrix (128-byte inner runs)
//   mode 1: box {128, 8} (512-byte inner runs), same 4 KB per store
//   mode 2: box {256, 4} over a [rows][256] matrix (1 KB inner runs)
// One CTA per SM, one thread issuing stores from a 64 KB SMEM ring (bulk_group depth D).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_store_rate profiles/tma_store_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int DEPTH>
__global__ void __launch_bounds__(32, 1)
store_rate(const __grid_constant__ CUtensorMap map, int64_t rows, int box_rows, int cols_el, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 16384; ++i) reinterpret_cast<float*>(sm)[i] = static_cast<float>(i);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int64_t tiles = rows / box_rows;
    for (int i = 0; i < iters; ++i) {
        const int64_t t = (blockIdx.x + static_cast<int64_t>(i) * gridDim.x) % tiles;
        const uint32_t src = smem_u32(sm) + (i % 16) * 4096;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                         reinterpret_cast<uint64_t>(&map)),
                     "r"(0), "r"(static_cast<int>(t * box_rows)), "r"(src)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH) : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
    const int64_t bytes = 4LL << 30;
    float* dst;
    if (cudaMalloc(&dst, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    for (int mode = 0; mode < 3; ++mode) {
        const int cols = mode == 2 ? 256 : 128;
        const int bx = mode == 0 ? 32 : mode == 1 ? 128 : 256;
        const int by = 1024 / bx;  // 4 KB per store
        const int64_t rows = bytes / (cols * 4);
        CUtensorMap map;
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 4)};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(by)};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dst, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", static_cast<int>(r)); continue; }
        // mode 0 walks 32-row boxes along a 128-column matrix: the box covers 32 rows x 128 B,
        // i.e. a quarter of each 512-byte row -- like the epilogue's warps; modes 1/2 write
        // whole rows.  Tiles index row blocks of `by` rows.
        for (int depth : {2, 8}) {
            const int iters = 4000;
            auto k = depth == 2 ? store_rate<2> : store_rate<8>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
            k<<<sms, 32, 65536>>>(map, rows, by, cols, iters);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<<<sms, 32, 65536>>>(map, rows, by, cols, iters);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("box {%3d, %2d} inner %4d B  depth %d  %7.0f GB/s  %s\n", bx, by, bx * 4, depth,
                   double(iters) * 4096 * sms / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
        }
    }
    cudaFree(dst);
    return 0;
}
