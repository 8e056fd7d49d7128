// Microbenchmark: TMA load rate of the forward Legendre GEMM's E/O operand boxes (B200).
// The E/O layout is eo[g][Rq][2F][4] fp32 (fft.cu FoldIO); a k-block of the A operand is
// 8 quads x 128 rows x 4 floats = 16 KB, 8 contiguous 2 KB runs.
//   mode 0: the GEMM's current 4D map, box {4, 128, 8, 1}: 16-byte inner dimension
//   mode 1: the same bytes and SMEM image as a 4D map with a 1 KB inner dimension,
//           dims {256, 2F*4/256, Rq, G}, box {256, 2, 8, 1}
//   mode 2: reference 2D box {32 fp32 (128 B, SWIZZLE_128B), 128 rows} (tma_rate.cu mode 0)
// One CTA per SM, one thread keeping S loads in flight; ~4 GB source (HBM-resident).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_eo_rate profiles/tma_eo_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int TWO_F = 2048, RQ = 96, G = 1300, KB = RQ / 8;  // 12 k-blocks per tile

template <int MODE>
__global__ void __launch_bounds__(32, 1)
eo_rate(const __grid_constant__ CUtensorMap map, int stages, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[16];
    constexpr uint32_t stage_bytes = 16384;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    constexpr int64_t mt = TWO_F / 128;
    const int64_t tiles = static_cast<int64_t>(G) * mt;
    auto issue = [&](int i, int s) {
        const int64_t tile = (blockIdx.x + static_cast<int64_t>(i / KB) * gridDim.x) % tiles;
        const int kb = i % KB;
        const int g = static_cast<int>(tile / mt), m = static_cast<int>(tile % mt);
        const uint32_t b = smem_u32(&bar[s]);
        const uint32_t dst = smem_u32(sm) + s * stage_bytes;
        const uint64_t mp = reinterpret_cast<uint64_t>(&map);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(stage_bytes));
        if (MODE == 0) {
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
                         "l"(mp), "r"(0), "r"(m * 128), "r"(kb * 8), "r"(g), "r"(b) : "memory");
        } else if (MODE == 1) {
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
                         "l"(mp), "r"(0), "r"(m * 2), "r"(kb * 8), "r"(g), "r"(b) : "memory");
        } else {
            // [G*Rq*2F/... rows x 384 cols] 2D view: same walk over 16 KB boxes
            const int row = static_cast<int>((tile * 128) % (static_cast<int64_t>(G) * RQ * TWO_F * 4 / 384 - 128));
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
                         "l"(mp), "r"(kb * 32), "r"(row), "r"(b) : "memory");
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
    long long* d_out;
    cudaMalloc(&d_out, sms * sizeof(long long));
    const int64_t elems = static_cast<int64_t>(G) * RQ * TWO_F * 4;
    float* src;
    if (cudaMalloc(&src, elems * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(src, 0, elems * 4);
    printf("source %.2f GB, %d SMs\n", elems * 4.0 / 1e9, sms);
    for (int mode = 0; mode < 3; ++mode) {
        CUtensorMap map;
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r;
        if (mode == 0) {
            cuuint64_t dims[4] = {4, TWO_F, RQ, G};
            cuuint64_t strides[3] = {16, 16ull * TWO_F, 16ull * TWO_F * RQ};
            cuuint32_t box[4] = {4, 128, 8, 1};
            r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else if (mode == 1) {
            cuuint64_t dims[4] = {256, TWO_F * 4 / 256, RQ, G};
            cuuint64_t strides[3] = {1024, 16ull * TWO_F, 16ull * TWO_F * RQ};
            cuuint32_t box[4] = {256, 2, 8, 1};
            r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            const int64_t rows = elems / 384;
            cuuint64_t dims[2] = {384, static_cast<cuuint64_t>(rows)};
            cuuint64_t strides[1] = {384 * 4};
            cuuint32_t box[2] = {32, 128};
            r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("mode %d: encode failed %d\n", mode, static_cast<int>(r)); continue; }
        for (int stages : {2, 4, 8}) {
            const int smem = stages * 16384;
            const int iters = 3000;
            auto k = mode == 0 ? eo_rate<0> : mode == 1 ? eo_rate<1> : eo_rate<2>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k<<<sms, 32, smem>>>(map, stages, iters, d_out);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<<<sms, 32, smem>>>(map, stages, iters, d_out);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double gbs = double(iters) * 16384 * sms / (ms * 1e-3) / 1e9;
            printf("%-22s stages %d  in-flight %3d KB/SM  %7.0f GB/s  %s\n",
                   mode == 0 ? "eo box {4,128,8,1}" : mode == 1 ? "eo box {256,2,8,1}" : "2D box {32,128} sw128",
                   stages, smem / 1024, gbs, cudaGetErrorString(err));
        }
    }
    cudaFree(src);
    return 0;
}
