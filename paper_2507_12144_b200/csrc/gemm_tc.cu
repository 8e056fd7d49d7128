// tcgen05 / TMEM / TMA grouped GEMM for sm_100a with a 3xTF32 precision split.
//
// Persistent, warp-specialised, one CTA (or CTA pair) per SM:
//   warp 0        TMA producer: A tile (data, fp32), B_hi and B_lo tiles (table) per stage
//   warp 1        MMA issuer (one elected thread): per K=8 step
//                   D += A_hi*B_hi ; D += A_hi*B_lo ; D += A_lo*B_hi   (kind::tf32)
//   warp 2        TMEM allocator
//   warps 4..7    converter: ALO -> A_lo = A - trunc_tf32(A) into TMEM (tcgen05.st), A_hi
//                 is the fp32 tile itself (see the kernel comment); otherwise A_hi/A_lo
//                 rna-split in SMEM
//   warps 8..     epilogue (4, or 8 in the pair variant): TMEM -> registers (pipelined
//                 tcgen05.ld 32x32b.x32) -> global, row-major through a per-warp SMEM
//                 transpose or column-major
// Pipelines: SMEM ring (full -> converted -> empty) and a double-buffered TMEM
// accumulator (full/empty) so the epilogue of tile i overlaps the MMAs of tile i+1.
// Operand tiles are K-major, SWIZZLE_64B (BK = 16) or SWIZZLE_128B (BK = 32, ALO).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>
#include <cstring>
#include <mutex>

#include "gemm.cuh"

namespace sph {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 16;               // fp32 per 64-byte swizzle row (SWIZZLE_64B variants)
constexpr int BK_ALO = 32;           // fp32 per 128-byte swizzle row (ALO variant, SWIZZLE_128B)
template <bool ALO> constexpr int bk_of() { return ALO ? BK_ALO : BK; }
// warps: 0 producer, 1 MMA, 2 TMEM allocator, 3 idle, 4..7 converter, 8.. epilogue
// (4 warps, or 8 = two per TMEM lane quarter splitting the columns in the pair variant)
// 8 epilogue warps (two per TMEM lane quarter) except the single-CTA Legendre variant,
// whose 3 x 64 KB ring leaves SMEM for only 4 warps' TMA-store staging
template <bool ALO, bool PAIR> constexpr int epi_warps() { return (ALO && !PAIR) ? 4 : 8; }
template <bool ALO, bool PAIR> constexpr int nthreads() { return (8 + epi_warps<ALO, PAIR>()) * 32; }


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ float gelu_erfc_dev(float x) {  // model.hpp:42-44
    // x * 0.5 * erfc(-x / sqrt 2) evaluated as 0.5 x (1 + erf(x / sqrt 2)): the same value up
    // to fp32 rounding (absolute error ~1e-8 where erfc's relative accuracy for very negative
    // x stops mattering) at a fraction of erfcf's instructions -- the MLP1 epilogue and the
    // GeLU transpose were issue-bound on it (cfg4 block pair 6.65 -> 6.25 ms,
    // profiles/r2/gelu_erf_ab.log).  -DSPH_GELU_ERFC restores the erfc form.
#ifdef SPH_GELU_ERFC
    return x * 0.5f * erfcf(-x * 0.70710678118654752440f);
#else
    const float h = 0.5f * x;
    return fmaf(h, erff(x * 0.70710678118654752440f), h);
#endif
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Barrier wait.  Debug builds (SPH_DEBUG=1 python paper_2507_12144_b200/build.py defines
// SPH_GEMM_WATCHDOG) bound it: a protocol bug then prints the barrier state and traps after
// 3 s instead of hanging.  Release builds spin without the bound, so a correct kernel
// preempted or time-sliced for longer than that is never killed.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
#ifdef SPH_GEMM_WATCHDOG
    uint64_t t0 = 0;
#endif
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
#ifdef SPH_GEMM_WATCHDOG
        const uint64_t t = global_ns();
        if (t0 == 0) t0 = t;
        else if (t - t0 > 3000000000ull) {
            uint64_t raw;
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(raw) : "r"(bar));
            if ((threadIdx.x & 31) == 0)
                printf("sph gemm watchdog: block %d warp %d barrier 0x%x parity %u raw 0x%016llx\n",
                       blockIdx.x, threadIdx.x / 32, bar, parity, static_cast<unsigned long long>(raw));
            __trap();
        }
#endif
    }
}
// arrive on the barrier at the same SMEM offset in cluster CTA `cta` (default .release.cta
// semantics, as CUTLASS's ClusterBarrier::arrive; .release.cluster measured ~2k cycles)
__device__ __forceinline__ void mbar_arrive_cta(uint32_t bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(bar), "r"(cta)
        : "memory");
}
// CTA-pair TMA: data lands in this CTA's SMEM, completion is signalled on the pair
// leader's barrier (same offset, peer bit cleared)
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar & 0xFEFFFFFFu)
        : "memory");
}
// L2 cache-policy variants (SPH_GEMM_L2HINT): evict-first for the streamed output, evict-
// last for the table tiles every M-run of a group re-reads
__device__ __forceinline__ uint64_t l2_policy(bool evict_last) {
    uint64_t pol;
    if (evict_last)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_2d_pair_hint(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                                      uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar & 0xFEFFFFFFu), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tc_commit_pair_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar), "h"(mask)
        : "memory");
}
// M = 256 over the CTA pair: rows 0..127 from the leader's A (SMEM or TMEM), 128..255
// from the peer's (same address); the B columns are split in halves between the two
// CTAs' SMEM (same offset)
__device__ __forceinline__ void tc_mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                    uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2,
                                             int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void tma_store_4d_hint(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2,
                                                  int c3, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_3d_hint(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2,
                                                  uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(src), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
// TMA tensor store of a [1][32][32] box from SMEM (bulk async-group of this thread)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                               uint32_t bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
// A operand from TMEM ("TS"): D += A[tmem] * B[smem]
__device__ __forceinline__ void tc_mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
        : "memory");
}
// 32 lanes x 32 bit, 32 consecutive columns per lane, asynchronous: the registers are
// valid only after tmem_wait32 on the same array (which takes them as "+r" operands so
// the compiler cannot move their uses above the wait)
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait32(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                   "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]),
                   "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]),
                   "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]),
                   "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]),
                   "+r"(r[31])
                 :
                 : "memory");
}
// UMMA shared-memory descriptor: K-major, rows of KB fp32 (64 B -> SWIZZLE_64B, layout 4;
// 128 B -> SWIZZLE_128B, layout 2), 8-row atoms (SBO = 8 rows), version 1.
template <int KB>
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
    static_assert(KB == 16 || KB == 32, "row width");
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);          // start address
    d |= static_cast<uint64_t>(1) << 16;                          // LBO (unused, swizzled K-major)
    d |= static_cast<uint64_t>((8 * KB * 4) >> 4) << 32;          // SBO: 8-row group stride
    d |= static_cast<uint64_t>(1) << 46;                          // descriptor version (sm100)
    d |= static_cast<uint64_t>(KB == 32 ? 2 : 4) << 61;           // SWIZZLE_128B / _64B
    return d;
}
// UMMA descriptor for the quad-interleaved A tile (SWIZZLE_NONE K-major): core matrix =
// 8 rows x 16 B contiguous, 8-row groups 128 B apart (SBO), k-quads 128 rows x 16 B =
// 2 KB apart (LBO); the TMA box [8 quads][128 rows][4] lands exactly in this layout.
__device__ __forceinline__ uint64_t make_sdesc_quad(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(2048 >> 4) << 16;  // LBO: next k-quad
    d |= static_cast<uint64_t>(128 >> 4) << 32;   // SBO: next 8-row group
    d |= static_cast<uint64_t>(1) << 46;
    return d;                                     // layout type 0 = SWIZZLE_NONE
}
// Instruction descriptor: kind::tf32, D f32, A/B tf32, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t make_idesc(int n, int m = BM) {  // m = 256: CTA pair
    uint32_t d = 0;
    d |= 1u << 4;                             // D format f32
    d |= 2u << 7;                             // A format tf32
    d |= 2u << 10;                            // B format tf32
    d |= static_cast<uint32_t>(n >> 3) << 17; // N >> 3
    d |= static_cast<uint32_t>(m >> 4) << 24; // M >> 4
    return d;
}

// KS (ALO only): 32-wide SWIZZLE_128B atoms per pipeline stage.  The loads, conversions
// and MMAs of a stage run per atom; its barrier waits, fences and commit once per stage.
template <int BN, int STAGES, bool ALO = false, bool PAIR = false, int KS = 1>
struct Smem {
    static constexpr int A_ATOM = BM * bk_of<ALO>() * 4;
    static constexpr int B_ATOM = (PAIR ? BN / 2 : BN) * bk_of<ALO>() * 4;  // PAIR: half
    static constexpr int A_TILE_BYTES = KS * A_ATOM;
    static constexpr int B_TILE_BYTES = KS * B_ATOM;
    static constexpr int A_BYTES = ALO ? A_TILE_BYTES : 2 * A_TILE_BYTES;  // A or (A_hi, A_lo)
    static constexpr int STAGE_BYTES = A_BYTES + 2 * B_TILE_BYTES;
    static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
    // full[S], conv[S], empty[S], tfull[2], tempty[2], tmem slot
    static constexpr int TILE_OFF = (BAR_OFF + (3 * STAGES + 4) * 8 + 16 + 1023) / 1024 * 1024;
    // epilogue staging: ALO -> two 4 KB TMA-store buffers per epilogue warp (also fits the
    // 32x33 transpose tiles of the plain-store fallback); else the transpose tiles
    // per-warp 32 x 32 transpose tiles (XOR-swizzled, no padding column)
    static constexpr int OUT_BYTES = ALO ? epi_warps<ALO, PAIR>() * 8192 : epi_warps<ALO, PAIR>() * 32 * 32 * 4;
    static constexpr int TOTAL = TILE_OFF + OUT_BYTES + 1024;  // + align slack
};

// CL > 1: thread-block cluster of CL CTAs on CL consecutive M-tiles of one (group,
// N-tile); each CTA TMA-loads 1/CL of the table tile and multicasts it to the whole
// cluster, so the L2 -> SMEM table traffic per CTA drops by CL.  A stage is refilled
// only after all CL consumers released it (multicast tcgen05.commit, count CL).
//
// ALO (the production variant): kind::tf32 reads fp32 operands and ignores the low 13
// mantissa bits, so the TMA-landed fp32 A tile IS A_hi = trunc_tf32(A) for the SMEM
// ("SS") MMAs A*B_hi and A*B_lo.  The converter warps only form A_lo = A -
// trunc_tf32(A) (exact) and tcgen05.st it into TMEM for the A_lo*B_hi ("TS") MMAs.
// K-block = 32 fp32 (SWIZZLE_128B rows): 12 MMAs per stage barrier round.  Measured with
// SPH_GEMM_TRACE / SPH_GEMM_DEBUG at BK = 16: ~950-1200 cycles per k-block at ANY tile N
// and ~700 even with the MMAs, converter, epilogue and table loads all disabled, i.e.
// the per-stage barrier round trip (producer -> TMA -> full -> convert -> MMA -> commit ->
// empty) and not the tensor pipe (6 MMAs = 576 cycles at N = 192, profiles/mma_rate.cu)
// bounded it; doubling the MMA work per round halves that cost per flop.  TMEM: 2 x BN
// accumulators + STAGES x 32 A_lo columns (384 + 96).
//
// PAIR (ALO, CL = 2): the cluster's two CTAs form one cta_group::2 MMA of M = 256.  Each
// CTA loads its own 128 data rows and HALF of the table tile (ninst/2 rows at n0 + rank *
// ninst/2), so per SM and k-block the inbound bytes drop from A + B to A + B/2 -- the
// measured limit of the single-CTA variant above.  The leader (rank 0) issues the MMAs
// (both CTAs' A / A_lo / B halves are read at the same SMEM / TMEM offsets); its full
// barrier also counts the peer's table-half bytes (.cta_group::2 TMA), its conv / tempty
// barriers take the peer's converter / epilogue arrivals (count 256), and its commits
// multicast to both CTAs' empty / tfull barriers.
template <int BN, int STAGES, int CL, bool ALO, bool PAIR = false, int KS = 1>
__global__ void __launch_bounds__(nthreads<ALO, PAIR>(), 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_bhi,
                   const __grid_constant__ CUtensorMap map_blo, const __grid_constant__ CUtensorMap map_d,
                   const GemmWork* __restrict__ works,
                   int ntiles, float* __restrict__ D,
                   int store_mode, int three_pass, long long* __restrict__ trace, int dbg,
                   int tma_store, int a_quad,  // a_quad: 0 2D SW128, 1 quad 16 B, 2 quad 512 B, 3 quad 1 KB
                   int d_mode, int d_t, int d_g2, int pf, GemmEpi epi, int l2hint, int blo_conv) {
    // dbg (diagnostic, SPH_GEMM_DEBUG bits; results are wrong when set): 1 epilogue skips
    // TMEM loads + stores, 2 converter skips its work, 4 no MMAs, 8 no table loads
    // (a whole-tile cp.async.bulk.prefetch.L2 one tile ahead was measured slower: cfg2
    // Legendre fwd / inv 5.07M / 4.65M vs 4.44M / 3.81M cycles without)
    // trace (diagnostic, SPH_GEMM_TRACE): CTA 0 records clock64 per k-block j < TR_N at
    // [0] producer issue, [1] data landed (converter wake), [2] converted, [3] MMA issue,
    // and per tile [4*TR_N + 2*lt] MMA start clock, [.. + 1] ninst * 1000 + k-blocks
    constexpr int TR_N = 512;
    const int tr_off = dbg >> 8;  // k-block window start (SPH_GEMM_DEBUG high bits)
    const bool tr = trace != nullptr && blockIdx.x == 0;
    using L = Smem<BN, STAGES, ALO, PAIR, KS>;
    static_assert(!PAIR || (ALO && CL == 2 && BN % 32 == 0), "pair mode: ALO, cluster of 2");
    static_assert(KS == 1 || ALO, "multi-atom stages: ALO variant");
    constexpr int KB = bk_of<ALO>();   // atom width (fp32 of K)
    constexpr int KST = KB * KS;       // K per pipeline stage
    constexpr int A_TILE_BYTES = L::A_TILE_BYTES;
    static_assert(!ALO || 2 * BN + STAGES * KST <= 512, "TMEM budget");
    constexpr uint32_t TMEM_COLS = ALO ? 512 : 2 * BN;
    extern __shared__ uint8_t smem_raw[];
    // 1 KB alignment by pointer arithmetic on the __shared__ array (keeps the shared
    // address space, so the epilogue tile accesses compile to LDS/STS)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    auto a_hi = [&](int s) { return sbase + s * L::STAGE_BYTES; };
    auto a_lo = [&](int s) { return sbase + s * L::STAGE_BYTES + A_TILE_BYTES; };
    auto b_hi = [&](int s) { return sbase + s * L::STAGE_BYTES + L::A_BYTES; };
    auto b_lo = [&](int s) { return sbase + s * L::STAGE_BYTES + L::A_BYTES + L::B_TILE_BYTES; };
    const uint32_t bars = sbase + L::BAR_OFF;
    auto full_bar = [&](int s) { return bars + 8 * s; };
    auto conv_bar = [&](int s) { return bars + 8 * (STAGES + s); };
    auto empty_bar = [&](int s) { return bars + 8 * (2 * STAGES + s); };
    auto tfull_bar = [&](int a) { return bars + 8 * (3 * STAGES + a); };
    auto tempty_bar = [&](int a) { return bars + 8 * (3 * STAGES + 2 + a); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::BAR_OFF + (3 * STAGES + 4) * 8);
    float* stile = reinterpret_cast<float*>(smem + L::TILE_OFF);  // epilogue transpose tiles

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint64_t pol_first = l2hint ? l2_policy(false) : 0, pol_last = l2hint ? l2_policy(true) : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar(s), 1);
            // PAIR: one aggregated arrival per CTA (named barrier + elected thread; 128
            // individual remote arrivals per stage cost ~2k cycles on the critical path)
            mbar_init(conv_bar(s), PAIR ? 2 : 128);
            mbar_init(empty_bar(s), PAIR ? 1 : CL);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar(a), 1);
            mbar_init(tempty_bar(a), PAIR ? 2 : epi_warps<ALO, PAIR>() * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
    }
    if (warp == 2) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    auto tmem_alo = [&](int s) { return tmem_base + 2 * BN + s * KST; };
    const int crank = CL > 1 ? static_cast<int>(cluster_rank()) : 0;
    const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    const uint16_t cmask = static_cast<uint16_t>((1u << CL) - 1);
    constexpr int B_ROWS = PAIR ? BN / 2 : BN / CL;  // table rows loaded by this CTA
    // PAIR: instruction N = N rounded up to 32; the peer's half starts at ninst / 2
    auto pair_half = [](const GemmWork& w) { return (w.nrem + 31) / 32 * 16; };
    // atom ka (K offset ka * KB) of the data tile into atom slot a of stage s
    auto load_a1 = [&](int s, int a, const GemmWork& w, int ka) {
        const uint32_t dst = a_hi(s) + a * L::A_ATOM;
        if (ALO && a_quad == 3)  // wider map: 64-row blocks of 1 KB
            tma_load_4d(dst, &map_a, 0, (w.m0 + crank * BM) / 64, ka * (KB / 4), w.ag, full_bar(s));
        else if (ALO && a_quad == 2)  // wide map: 32-row blocks of 512 B
            tma_load_4d(dst, &map_a, 0, (w.m0 + crank * BM) / 32, ka * (KB / 4), w.ag, full_bar(s));
        else if (ALO && a_quad)
            tma_load_4d(dst, &map_a, 0, w.m0 + crank * BM, ka * (KB / 4), w.ag, full_bar(s));
        else
            tma_load_2d(dst, &map_a, ka * KB, w.a_row + crank * BM, full_bar(s));
    };
    // atoms of stage k-block kb that hold K (the last stage of a tile may be partial)
    auto natoms_of = [&](const GemmWork& w, int kb) { return min(KS, (w.K - kb * KST + KB - 1) / KB); };
    auto load_a = [&](int s, const GemmWork& w, int kb, int na) {
        for (int a = 0; a < na; ++a) load_a1(s, a, w, kb * KS + a);
    };
    // L2 prefetch of a data tile k-block (same box as load_a)
    auto prefetch_a = [&](const GemmWork& w, int kb) {
        if (ALO && a_quad == 3)
            tma_prefetch_4d(&map_a, 0, (w.m0 + crank * BM) / 64, kb * (KB / 4), w.ag);
        else if (ALO && a_quad == 2)
            tma_prefetch_4d(&map_a, 0, (w.m0 + crank * BM) / 32, kb * (KB / 4), w.ag);
        else if (ALO && a_quad)
            tma_prefetch_4d(&map_a, 0, w.m0 + crank * BM, kb * (KB / 4), w.ag);
        else
            tma_prefetch_2d(&map_a, kb * KB, w.a_row + crank * BM);
    };
    // operands of k-step kk (8 fp32 of K) of a stage: atom kk / 4, 32-byte step kk % 4
    // (quad layout: the atoms' k-quads are contiguous 2 KB blocks)
    auto adesc = [&](int s, int kk) {
        if (ALO && a_quad) return make_sdesc_quad(a_hi(s) + kk * 2 * 2048);
        if constexpr (KS == 1) return make_sdesc<KB>(a_hi(s) + kk * 32);  // one atom: no split
        return make_sdesc<KB>(a_hi(s) + (kk / (KB / 8)) * L::A_ATOM + (kk % (KB / 8)) * 32);
    };
    auto bdesc = [&](uint32_t base, int kk) {
        if constexpr (KS == 1) return make_sdesc<KB>(base + kk * 32);
        return make_sdesc<KB>(base + (kk / (KB / 8)) * L::B_ATOM + (kk % (KB / 8)) * 32);
    };
    // each role walks tiles cid, cid + ncl, ... and loads the next descriptor one tile ahead
    GemmWork wnext{};
    if (cid < ntiles) wnext = works[cid];
    auto next_work = [&](int t) {
        const GemmWork w = wnext;
        if (t + ncl < ntiles) wnext = works[t + ncl];
        return w;
    };
    if (CL > 1) cluster_sync_all();  // peers' barriers initialised before any multicast

    if (warp == 0) {
        // ------------------------------------------------------------- producer
        if (lane == 0) {
            int s = 0, j = 0;
            uint32_t ph = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                const GemmWork w = next_work(t);
                const int nkb = (w.K + KST - 1) / KST;
                const bool has_next = t + ncl < ntiles;
                const GemmWork wn = wnext;  // next tile's descriptor (loaded a tile ahead)
                const int nkb_n = (wn.K + KST - 1) / KST;
                for (int kb = 0; kb < nkb; ++kb, ++j) {
                    // data-tile L2 prefetch pf k-blocks ahead (HBM latency dominates the
                    // ring's round trip; SMEM and TMEM allow no further stages)
                    if (pf > 0) {
                        const int kp = kb + pf;
                        if (kp < nkb)
                            prefetch_a(w, kp * KS);
                        else if (has_next && kp - nkb < nkb_n)
                            prefetch_a(wn, (kp - nkb) * KS);
                    }
                    mbar_wait(empty_bar(s), ph ^ 1);
                    if (tr && j >= tr_off && j - tr_off < TR_N) trace[j - tr_off] = clock64();
                    const int na = natoms_of(w, kb);
                    if (dbg & 8) {
                        mbar_expect_tx(full_bar(s), na * L::A_ATOM);
                        load_a(s, w, kb, na);
                        if (++s == STAGES) { s = 0; ph ^= 1; }
                        continue;
                    }
                    if (PAIR && three_pass && blo_conv) {
                        // converter-split table: each CTA's converter must see ITS table half
                        // land, so both halves signal their own CTA's full barrier (plain TMA);
                        // the leader's MMA still waits for both through the conv barrier
                        mbar_expect_tx(full_bar(s), na * (L::A_ATOM + L::B_ATOM));
                        load_a(s, w, kb, na);
                        const int brow = w.b_row + crank * pair_half(w);
                        for (int a = 0; a < na; ++a)
                            tma_load_2d(b_hi(s) + a * L::B_ATOM, &map_bhi, (kb * KS + a) * KB, brow, full_bar(s));
                        if (++s == STAGES) { s = 0; ph ^= 1; }
                        continue;
                    }
                    if constexpr (PAIR) {
                        // leader's full barrier: own A + both CTAs' table halves; peer's: A
                        const int nb = (three_pass ? 2 : 1) * na * L::B_ATOM;
                        mbar_expect_tx(full_bar(s), na * L::A_ATOM + (crank == 0 ? 2 * nb : 0));
                        load_a(s, w, kb, na);
                        const int brow = w.b_row + crank * pair_half(w);
                        for (int a = 0; a < na; ++a) {
                            const int kx = (kb * KS + a) * KB;
                            if (l2hint & 2) {
                                tma_load_2d_pair_hint(b_hi(s) + a * L::B_ATOM, &map_bhi, kx, brow, full_bar(s), pol_last);
                                if (three_pass)
                                    tma_load_2d_pair_hint(b_lo(s) + a * L::B_ATOM, &map_blo, kx, brow, full_bar(s),
                                                          pol_last);
                                continue;
                            }
                            tma_load_2d_pair(b_hi(s) + a * L::B_ATOM, &map_bhi, kx, brow, full_bar(s));
                            if (three_pass)
                                tma_load_2d_pair(b_lo(s) + a * L::B_ATOM, &map_blo, kx, brow, full_bar(s));
                        }
                        if (++s == STAGES) { s = 0; ph ^= 1; }
                        continue;
                    }
                    mbar_expect_tx(full_bar(s), na * (L::A_ATOM + (three_pass && !blo_conv ? 2 : 1) * L::B_ATOM));
                    load_a(s, w, kb, na);
                    for (int a = 0; a < na; ++a) {
                        const int kx = (kb * KS + a) * KB;
                        if (CL == 1) {
                            tma_load_2d(b_hi(s) + a * L::B_ATOM, &map_bhi, kx, w.b_row, full_bar(s));
                            if (three_pass && !blo_conv)
                                tma_load_2d(b_lo(s) + a * L::B_ATOM, &map_blo, kx, w.b_row, full_bar(s));
                        } else {
                            const uint32_t off = a * L::B_ATOM + crank * B_ROWS * KB * 4;
                            tma_load_2d_mc(b_hi(s) + off, &map_bhi, kx, w.b_row + crank * B_ROWS, full_bar(s),
                                           cmask);
                            if (three_pass && !blo_conv)
                                tma_load_2d_mc(b_lo(s) + off, &map_blo, kx, w.b_row + crank * B_ROWS,
                                               full_bar(s), cmask);
                        }
                    }
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA issuer
        if (lane == 0 && (!PAIR || crank == 0)) {
            int s = 0, j = 0;
            uint32_t ph = 0;
            int lt = 0;
            for (int t = cid; t < ntiles; t += ncl, ++lt) {
                const GemmWork w = next_work(t);
                const int nkb = (w.K + KST - 1) / KST;
                const int acc = lt & 1;
                const uint32_t aph = (lt >> 1) & 1;
                const int nrem = w.nrem;
                const int ninst = PAIR ? (nrem + 31) / 32 * 32 : (nrem + 15) / 16 * 16;
                const uint32_t idesc = make_idesc(ninst, PAIR ? 2 * BM : BM);
                const uint32_t tmem_d = tmem_base + acc * BN;
                mbar_wait(tempty_bar(acc), aph ^ 1);
                tc_fence_after();
                if (tr && lt < 2048) {
                    trace[4 * TR_N + 2 * lt] = clock64();
                    trace[4 * TR_N + 2 * lt + 1] = ninst * 1000 + nkb;
                }
                for (int kb = 0; kb < nkb; ++kb, ++j) {
                    mbar_wait(conv_bar(s), ph);  // converter waited full(s): data landed + A_lo
                    tc_fence_after();
                    if (tr && j >= tr_off && j - tr_off < TR_N) trace[3 * TR_N + j - tr_off] = clock64();
                    const int ksteps = (dbg & 4) ? 0 : min(KST / 8, (w.K - kb * KST + 7) / 8);
                    for (int kk = 0; kk < ksteps; ++kk) {
                        const uint64_t ahi = adesc(s, kk);
                        const uint64_t bhi = bdesc(b_hi(s), kk);
                        if constexpr (PAIR) {
                            tc_mma_tf32_pair(tmem_d, ahi, bhi, idesc, (kb | kk) ? 1u : 0u);
                            if (three_pass) {
                                tc_mma_tf32_pair(tmem_d, ahi, bdesc(b_lo(s), kk), idesc, 1u);
                                tc_mma_tf32_ts_pair(tmem_d, tmem_alo(s) + kk * 8, bhi, idesc, 1u);
                            }
                            continue;
                        }
                        tc_mma_tf32(tmem_d, ahi, bhi, idesc, (kb | kk) ? 1u : 0u);
                        if (three_pass) {
                            tc_mma_tf32(tmem_d, ahi, bdesc(b_lo(s), kk), idesc, 1u);
                            if constexpr (ALO)
                                tc_mma_tf32_ts(tmem_d, tmem_alo(s) + kk * 8, bhi, idesc, 1u);
                            else
                                tc_mma_tf32(tmem_d, make_sdesc<KB>(a_lo(s) + kk * 32), bhi, idesc, 1u);
                        }
                    }
                    if (PAIR)
                        tc_commit_pair_mc(empty_bar(s), cmask);
                    else if (CL == 1)
                        tc_commit(empty_bar(s));
                    else
                        tc_commit_mc(empty_bar(s), cmask);
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
                if (PAIR)
                    tc_commit_pair_mc(tfull_bar(acc), cmask);
                else
                    tc_commit(tfull_bar(acc));
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ----------------------------------------------------------- converter
        const int ct = threadIdx.x - 128;
        int s = 0, j = 0;
        uint32_t ph = 0;
        const bool trc = tr && (ct & 127) == 0;
        for (int t = cid; t < ntiles; t += ncl) {
            const GemmWork w = next_work(t);
            const int nkb = (w.K + KST - 1) / KST;
            for (int kb = 0; kb < nkb; ++kb, ++j) {
                mbar_wait(full_bar(s), ph);
                if (trc && j >= tr_off && j - tr_off < TR_N) trace[TR_N + j - tr_off] = clock64();
                if constexpr (ALO) {
                    if (three_pass && !(dbg & 2)) {
                        // this warp owns TMEM lanes 32q..32q+31 = tile rows; read the row's
                        // 32 fp32 from the SWIZZLE_128B tile (16-byte chunk c of row r sits
                        // at chunk c ^ (r & 7): conflict-free for 8 consecutive rows)
                        const int q = warp & 3;
                        const int row = 32 * q + lane;
                        const int na = natoms_of(w, kb);
                        for (int at = 0; at < na; ++at) {
                        const float4* rowp = reinterpret_cast<const float4*>(smem + (a_hi(s) - sbase) +
                                                                             at * L::A_ATOM + row * KB * 4);
                        const float4* quadp =
                            reinterpret_cast<const float4*>(smem + (a_hi(s) - sbase) + at * L::A_ATOM) + row;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            float lo[16];
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                // quad layout: k-quad (4h + c) of the row at quad * 2 KB + row * 16 B
                                const float4 v = a_quad ? quadp[(4 * h + c) * BM] : rowp[(4 * h + c) ^ (row & 7)];
                                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    lo[4 * c + e] = vv[e] - __uint_as_float(__float_as_uint(vv[e]) & 0xFFFFE000u);
                            }
                            tmem_st16(tmem_alo(s) + at * KB + 16 * h + (static_cast<uint32_t>(32 * q) << 16), lo);
                        }
                        }
                        if (blo_conv) {
                            // the raw fp32 table tile split in place, element-wise at the same
                            // (swizzled) SMEM positions, exactly as the host split of the
                            // forward tables: hi = rna_tf32(B), lo = B - hi.  Runs while the
                            // TMEM stores drain; the async proxy (the MMA's descriptor reads)
                            // sees the generic stores after the proxy fence
                            float4* bh = reinterpret_cast<float4*>(smem + (b_hi(s) - sbase));
                            float4* bl = reinterpret_cast<float4*>(smem + (b_lo(s) - sbase));
                            const int nb4 = na * L::B_ATOM / 16;
                            for (int i = ct; i < nb4; i += 128) {
                                const float4 v = bh[i];
                                float4 h, o;
                                uint32_t u;
                                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v.x)); h.x = __uint_as_float(u);
                                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v.y)); h.y = __uint_as_float(u);
                                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v.z)); h.z = __uint_as_float(u);
                                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v.w)); h.w = __uint_as_float(u);
                                o.x = v.x - h.x;
                                o.y = v.y - h.y;
                                o.z = v.z - h.z;
                                o.w = v.w - h.w;
                                bh[i] = h;
                                bl[i] = o;
                            }
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        }
                        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                        tc_fence_before();
                    }
                } else if (three_pass) {
                    float4* hi = reinterpret_cast<float4*>(smem + (a_hi(s) - sbase));
                    float4* lo = reinterpret_cast<float4*>(smem + (a_lo(s) - sbase));
#pragma unroll
                    for (int i = 0; i < A_TILE_BYTES / 16 / 128; ++i) {
                        const int idx = ct + i * 128;
                        float4 v = hi[idx];
                        float4 h, l;
                        uint32_t u;
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v.x)); h.x = __uint_as_float(u);
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v.y)); h.y = __uint_as_float(u);
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v.z)); h.z = __uint_as_float(u);
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v.w)); h.w = __uint_as_float(u);
                        l.x = v.x - h.x; l.y = v.y - h.y; l.z = v.z - h.z; l.w = v.w - h.w;
                        hi[idx] = h;
                        lo[idx] = l;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                if (PAIR) {
                    // all 4 converter warps done (their tcgen05.st fenced) -> one arrival on
                    // the leader's conv barrier for this CTA
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (ct == 0) mbar_arrive_cta(conv_bar(s), 0);
                    // trace: global-timer stamps of both CTAs' conversions (cross-SM comparable)
                    if (trace != nullptr && blockIdx.x < 2 && ct == 0 && j >= tr_off && j - tr_off < TR_N)
                        trace[4 * TR_N + 4096 + blockIdx.x * TR_N + (j - tr_off)] = static_cast<long long>(global_ns());
                } else {
                    mbar_arrive(conv_bar(s));
                }
                if (trc && j >= tr_off && j - tr_off < TR_N) trace[2 * TR_N + j - tr_off] = clock64();
                if (++s == STAGES) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp >= 8) {
        // ------------------------------------------------------------- epilogue
        // warp (8 + i): TMEM lane quarter q = warp & 3 (rows 32q..32q+31), 32-column chunks
        // c = 32 * (i / 4) + 32 * EH * k; the next chunk's tcgen05.ld is in flight while
        // the current one is stored
        constexpr int EH = epi_warps<ALO, PAIR>() / 4;
        const int q = warp & 3;
        const int eh = (warp - 8) / 4;
        float* tile = stile + (warp - 8) * 32 * 32;  // per-warp 32x32 transpose (STORE_ROW),
                                                     // element (r, col) at r * 32 + (col ^ r)
        // TMA-store path (ALO): ping-pong 4 KB staging buffers per warp; lane 0 issues the
        // 3D tensor store of each 32 x 32 chunk and recycles a buffer after wait_group.read
        // TMA-store path: ALO kernels ping-pong two 4 KB staging buffers per warp; the
        // non-ALO row-store kernels (row_tma) use one (their SMEM ring leaves 4 KB per warp)
        const bool tstore = tma_store && (ALO || store_mode == STORE_ROW);
        uint8_t* obase = smem + L::TILE_OFF + (warp - 8) * (ALO ? 8192 : 4096);
        int nchunk = 0;
        int lt = 0;
        for (int t = cid; t < ntiles; t += ncl, ++lt) {
            const GemmWork w = next_work(t);
            const int acc = lt & 1;
            const uint32_t aph = (lt >> 1) & 1;
            const int nrem = w.nrem;
            mbar_wait(tfull_bar(acc), aph);
            tc_fence_after();
            const int row0 = w.m0 + crank * BM + q * 32;
            const uint32_t trow = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
            float* dbase = D + w.d_off;
            const int ncols = store_mode == STORE_ROW ? w.ncols : nrem;
            uint32_t va[32], vb[32];
            int c = 32 * eh;
            if (!(dbg & 1) && c < nrem) {
                tmem_ld32_async(trow + c, va);
                tmem_wait32(va);
            }
            for (; !(dbg & 1) && c < ncols; c += 32 * EH) {
                const int cn = c + 32 * EH;
                const bool more = cn < nrem;
                if (more) tmem_ld32_async(trow + cn, vb);
                if (tstore) {
                    float* ob = reinterpret_cast<float*>(obase + (ALO ? (nchunk & 1) * 4096 : 0));
                    if (ALO) {
                        if (lane == 0 && nchunk >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    } else {
                        if (lane == 0 && nchunk >= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    }
                    __syncwarp();
                    if (store_mode == STORE_ROW) {
                        // box {32 cols, 32 rows}, SWIZZLE_128B: row = lane, 16-byte chunk k of
                        // the row at k ^ (row & 7); fused bias + GeLU (epi mode 1) on the way
                        float4* orow = reinterpret_cast<float4*>(ob) + lane * 8;
                        if constexpr (ALO) {  // no fused epilogue in the A_lo-in-TMEM kernels
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                float e[4];
#pragma unroll
                                for (int x = 0; x < 4; ++x)
                                    e[x] = (c + 4 * k + x < nrem) ? __uint_as_float(va[4 * k + x]) : 0.f;
                                orow[k ^ (lane & 7)] = make_float4(e[0], e[1], e[2], e[3]);
                            }
                        } else {
                            float bv[32];
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) bv[jj] = 0.f;
                            if (epi.mode == 1) {
                                const float* bsrc = epi.bias + w.n0 + c;
                                if (c + 32 <= nrem && (reinterpret_cast<uintptr_t>(bsrc) & 15) == 0) {
#pragma unroll
                                    for (int q = 0; q < 8; ++q) {
                                        const float4 b4 = __ldg(reinterpret_cast<const float4*>(bsrc) + q);
                                        bv[4 * q] = b4.x;
                                        bv[4 * q + 1] = b4.y;
                                        bv[4 * q + 2] = b4.z;
                                        bv[4 * q + 3] = b4.w;
                                    }
                                } else {
#pragma unroll
                                    for (int jj = 0; jj < 32; ++jj) bv[jj] = c + jj < nrem ? __ldg(bsrc + jj) : 0.f;
                                }
                            }
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                float e[4];
#pragma unroll
                                for (int x = 0; x < 4; ++x) {
                                    const int jj = 4 * k + x;
                                    const float v = __uint_as_float(va[jj]);
                                    e[x] = (c + jj < nrem) ? (epi.mode == 1 ? gelu_erfc_dev(v + bv[jj]) : v) : 0.f;
                                }
                                orow[k ^ (lane & 7)] = make_float4(e[0], e[1], e[2], e[3]);
                            }
                        }
                    } else {
                        // box {32 rows m (contiguous), 32 cols n}: element (n = jj, m = lane)
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            ob[jj * 32 + lane] = (c + jj < nrem) ? __uint_as_float(va[jj]) : 0.f;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        if (l2hint & 1) {  // streamed output: evict-first
                            if (store_mode == STORE_ROW)
                                tma_store_3d_hint(&map_d, smem_u32(ob), w.n0 + c, row0, w.dg, pol_first);
                            else if (d_mode == 1)
                                tma_store_4d_hint(&map_d, smem_u32(ob), row0 % EOI_TILE, w.dg, row0 / EOI_TILE, w.n0 + c,
                                                  pol_first);
                            else
                                tma_store_3d_hint(&map_d, smem_u32(ob), row0, w.n0 + c, w.dg, pol_first);
                        } else if (store_mode == STORE_ROW)
                            tma_store_3d(&map_d, smem_u32(ob), w.n0 + c, row0, w.dg);
                        else if (d_mode == 1)  // box {32 rows of the field tile, group, tile, 32 n}
                            tma_store_4d(&map_d, smem_u32(ob), row0 % EOI_TILE, w.dg, row0 / EOI_TILE, w.n0 + c);
                        else
                            tma_store_3d(&map_d, smem_u32(ob), row0, w.n0 + c, w.dg);
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    ++nchunk;
                } else if (store_mode == STORE_ROW) {
                    // transpose through the per-warp 32 x 32 SMEM tile in 16-byte chunks:
                    // chunk q of row r sits at q ^ (r & 7) (conflict-free STS.128 by rows,
                    // LDS.128 by 8-lane row groups), stored as 4 rows of 128 coalesced bytes
                    // per STG.128 (the word-wise form issued 32 LDG + 32 STS + 32 LDS +
                    // 32 STG per chunk: the cfg4 MLP GEMM was epilogue-bound)
                    float4* t4 = reinterpret_cast<float4*>(tile);
                    float bv[32];
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) bv[jj] = 0.f;
                    if (epi.mode == 1) {  // fused bias + GeLU (erfc form); bias chunks are warp-uniform
                        const float* bsrc = epi.bias + w.n0 + c;
                        if (c + 32 <= nrem && (reinterpret_cast<uintptr_t>(bsrc) & 15) == 0) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 b4 = __ldg(reinterpret_cast<const float4*>(bsrc) + q);
                                bv[4 * q] = b4.x;
                                bv[4 * q + 1] = b4.y;
                                bv[4 * q + 2] = b4.z;
                                bv[4 * q + 3] = b4.w;
                            }
                        } else {
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) bv[jj] = c + jj < nrem ? __ldg(bsrc + jj) : 0.f;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float e[4];
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const int jj = 4 * q + x;
                            const float v = __uint_as_float(va[jj]);
                            e[x] = (c + jj < nrem) ? (epi.mode == 1 ? gelu_erfc_dev(v + bv[jj]) : v) : 0.f;
                        }
                        t4[lane * 8 + (q ^ (lane & 7))] = make_float4(e[0], e[1], e[2], e[3]);
                    }
                    __syncwarp();
                    const int qq = lane & 7;
                    const int colq = w.n0 + c + 4 * qq;
                    const bool vec = (w.ldd & 3) == 0 && (reinterpret_cast<uintptr_t>(dbase) & 15) == 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int r = 4 * k + (lane >> 3);
                        const int mr = row0 + r;
                        const float4 v = t4[r * 8 + (qq ^ (r & 7))];
                        if (mr >= w.M) continue;
                        float* dst = dbase + static_cast<int64_t>(mr) * w.ldd + colq;
                        if (vec && c + 4 * qq + 4 <= ncols) {
                            *reinterpret_cast<float4*>(dst) = v;
                        } else {
                            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int x = 0; x < 4; ++x)
                                if (c + 4 * qq + x < ncols) dst[x] = vv[x];
                        }
                    }
                    __syncwarp();
                } else {
                    const int m = row0 + lane;
                    if (m < w.M && d_mode == 1) {
                        float* dp = D + ((static_cast<int64_t>(w.n0 + c) * d_t + m / EOI_TILE) * d_g2 + w.dg) * EOI_TILE +
                                    (m % EOI_TILE);
                        const int64_t nstride = static_cast<int64_t>(d_t) * d_g2 * EOI_TILE;
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            if (c + jj < nrem) dp[jj * nstride] = __uint_as_float(va[jj]);
                    } else if (m < w.M && epi.mode == 2) {
                        // fused layer-scaled residual: D = res + scale[n] * (acc + bias[n])
                        // residual / scale / bias loads issued in groups of 8 before the
                        // group's stores (the compiler cannot move loads of res past stores
                        // to D, so one-at-a-time serialised ~32 HBM latencies per chunk)
                        const int64_t e0 = w.d_off + static_cast<int64_t>(w.n0 + c) * w.ldd + m;
#pragma unroll
                        for (int g8 = 0; g8 < 32; g8 += 8) {
                            float rv[8], sv[8], bv[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const int jj = g8 + u;
                                const bool ok = c + jj < nrem;
                                const int n = w.n0 + c + jj;
                                rv[u] = ok ? __ldg(epi.res + e0 + static_cast<int64_t>(jj) * w.ldd) : 0.f;
                                sv[u] = ok ? __ldg(epi.scale + n) : 0.f;
                                bv[u] = ok ? __ldg(epi.bias + n) : 0.f;
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const int jj = g8 + u;
                                if (c + jj < nrem)
                                    D[e0 + static_cast<int64_t>(jj) * w.ldd] =
                                        rv[u] + sv[u] * (__uint_as_float(va[jj]) + bv[u]);
                            }
                        }
                    } else if (m < w.M) {
                        float* dp = dbase + static_cast<int64_t>(w.n0 + c) * w.ldd + m;
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            if (c + jj < nrem) dp[static_cast<int64_t>(jj) * w.ldd] = __uint_as_float(va[jj]);
                    }
                }
                if (more) {
                    tmem_wait32(vb);
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) va[jj] = vb[jj];
                }
            }
            tc_fence_before();
            if (PAIR) {  // one aggregated arrival per CTA on the leader's tempty barrier
                asm volatile("bar.sync 2, %0;" ::"n"(epi_warps<ALO, PAIR>() * 32) : "memory");
                if (warp == 8 && lane == 0) mbar_arrive_cta(tempty_bar(acc), 0);
            } else {
                mbar_arrive(tempty_bar(acc));
            }
        }
        if (tstore && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }

    __syncthreads();
    if (CL > 1) cluster_sync_all();  // no CTA leaves while peers may still multicast into it
    if (warp == 2) {
        tc_fence_after();
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(TMEM_COLS)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(TMEM_COLS)
                         : "memory");
    }
}

// ------------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) fail(SPH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

static CUtensorMap make_map(const Mat2D& m, int box_rows, int kb) {
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    require(m.ld * 4 % 16 == 0, "gemm: operand row stride must be a multiple of 16 bytes");
    require((reinterpret_cast<uintptr_t>(m.p) & 15) == 0, "gemm: operand must be 16B aligned");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(m.cols), static_cast<cuuint64_t>(m.rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(m.ld * 4)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kb), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(m.p), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             kb == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(SPH_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return map;
}

// rows per inner run of the quad-interleaved A map: 64 (1 KB, SPH_GEMM_AQUAD_1K=1),
// 32 (512 B) or 1 (16-byte core-matrix rows) -- every A tile starts on a multiple of BM
static int quad_rows(const GroupedGemm& g) {
    static const bool k1 = [] {
        const char* e = std::getenv("SPH_GEMM_AQUAD_1K");
        return e && std::atoi(e) != 0;
    }();
    if (k1 && g.a_rows_g % 64 == 0) return 64;
    return g.a_rows_g % 32 == 0 ? 32 : 1;
}

template <int BN, int STAGES, int CL, bool ALO = false, bool PAIR = false, int KS = 1>
static void launch(const GroupedGemm& g, const float* A, const float* Bhi, const float* Blo,
                   float* D, bool three, cudaStream_t st, GemmEpi epi) {
    require(epi.mode == 0 || (!ALO && (epi.mode == 1) == (g.store == STORE_ROW)),
            "gemm: fused epilogue mode does not match the store mode / variant");
    using L = Smem<BN, STAGES, ALO, PAIR, KS>;
    static_assert(L::TOTAL <= 232448, "gemm: shared memory budget");
    auto kern = gemm_tf32x3_kernel<BN, STAGES, CL, ALO, PAIR, KS>;
    static int grid = 0;
    static std::once_flag once;
    std::call_once(once, [&] {
        SPH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
        grid = num_sms() / CL * CL;
        if (CL > 1) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(nthreads<ALO, PAIR>());
            cfg.dynamicSmemBytes = L::TOTAL;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = CL;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) == cudaSuccess && ncl > 0)
                grid = std::min(grid, ncl * CL);
        }
    });
    Mat2D am = g.A;
    am.p = A;
    CUtensorMap ma;
    const bool quad = ALO && g.a_quad;
    if (quad) {
        std::memset(&ma, 0, sizeof(ma));
        require((reinterpret_cast<uintptr_t>(A) & 15) == 0, "gemm: operand must be 16B aligned");
        // rows % 32 == 0: dims {32 rows x 4 (512 B contiguous), row blocks, quads, groups},
        // box {128, 4, 8, 1} -> 512-byte TMA requests; otherwise {4, rows, quads, groups}
        // with 16-byte requests (measured 3.1 vs 2.4 ms on the cfg2 forward GEMM)
        // rows % 64 == 0 (and SPH_GEMM_AQUAD_1K=1): 1 KB inner runs (64 rows x 4), the same
        // SMEM image (profiles/tma_eo_rate.cu: 16-byte inner boxes cap TMA at 3.8 TB/s)
        const int rb = quad_rows(g);
        const bool wide = rb > 1;
        cuuint64_t dims[4] = {wide ? 4u * rb : 4u,
                              static_cast<cuuint64_t>(wide ? g.a_rows_g / rb : g.a_rows_g),
                              static_cast<cuuint64_t>(g.a_kq), static_cast<cuuint64_t>(g.a_groups)};
        cuuint64_t strides[3] = {static_cast<cuuint64_t>(wide ? 16 * rb : 16), static_cast<cuuint64_t>(g.a_rows_g * 16),
                                 static_cast<cuuint64_t>(g.a_kq * g.a_rows_g * 16)};
        cuuint32_t box[4] = {wide ? 4u * rb : 4u, wide ? static_cast<cuuint32_t>(BM / rb) : static_cast<cuuint32_t>(BM),
                             static_cast<cuuint32_t>(bk_of<ALO>() / 4), 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = encode_fn()(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(A), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(SPH_ERR_CUDA, "cuTensorMapEncodeTiled (A quad) failed: " + std::to_string(r));
    } else {
        ma = make_map(am, BM, bk_of<ALO>());
    }
    Mat2D bh = g.Bhi, bl = g.Blo;
    bh.p = Bhi;
    bl.p = Blo;
    const CUtensorMap mbh = make_map(bh, PAIR ? BN / 2 : BN / CL, bk_of<ALO>());
    const CUtensorMap mbl = make_map(three ? bl : bh, PAIR ? BN / 2 : BN / CL, bk_of<ALO>());
    CUtensorMap md;
    std::memset(&md, 0, sizeof(md));
    const bool tstore = g.tma_store && (ALO || g.store == STORE_ROW);
    if (tstore && g.d_mode == 1) {
        // [n][field tile][group][EOI_TILE]: box {32, 1, 1, 32} = a warp's 128-byte quarter of
        // a 512-byte run, the CTA's 4 lane-quarter warps fill the run together (16-row tiles
        // with 64-byte pieces measured 3.5 vs 2.1 ms on the cfg2 inverse GEMM)
        cuuint64_t dims[4] = {EOI_TILE, static_cast<cuuint64_t>(g.d_g2), static_cast<cuuint64_t>(g.d_t),
                              static_cast<cuuint64_t>(g.d_rows)};
        cuuint64_t strides[3] = {4 * EOI_TILE, static_cast<cuuint64_t>(g.d_g2 * 4 * EOI_TILE),
                                 static_cast<cuuint64_t>(g.d_t * g.d_g2 * 4 * EOI_TILE)};
        cuuint32_t box[4] = {32, 1, 1, 32};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        require((reinterpret_cast<uintptr_t>(D) & 15) == 0, "gemm: output must be 16B aligned");
        CUresult r = encode_fn()(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, D, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(SPH_ERR_CUDA, "cuTensorMapEncodeTiled (D tiles) failed: " + std::to_string(r));
    } else if (tstore) {
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.d_ldd), static_cast<cuuint64_t>(g.d_rows),
                              static_cast<cuuint64_t>(g.d_groups3)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.d_ldd * 4),
                                 static_cast<cuuint64_t>(g.d_rows * g.d_ldd * 4)};
        cuuint32_t box[3] = {32, 32, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        require((reinterpret_cast<uintptr_t>(D) & 15) == 0, "gemm: output must be 16B aligned");
        CUresult r = encode_fn()(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, D, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 g.store == STORE_ROW ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(SPH_ERR_CUDA, "cuTensorMapEncodeTiled (D) failed: " + std::to_string(r));
    }
    const GemmTileList& tl = g.tiles_for(CL);
    int gsz = static_cast<int>(std::min<int64_t>(tl.n * CL, grid));
    if (gemm_sm_cap() > 0) gsz = std::min(gsz, gemm_sm_cap());
    gsz = std::max(CL, gsz / CL * CL);
    ProfScope prof(g.name, st, g.flops);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(gsz);
    cfg.blockDim = dim3(nthreads<ALO, PAIR>());
    cfg.dynamicSmemBytes = L::TOTAL;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = CL > 1 ? 1 : 0;
    static const char* trace_dir = std::getenv("SPH_GEMM_TRACE");  // diagnostic only
    static const int dbg = std::getenv("SPH_GEMM_DEBUG") ? std::atoi(std::getenv("SPH_GEMM_DEBUG")) : 0;
    static const int pf_env = std::getenv("SPH_GEMM_PF") ? std::atoi(std::getenv("SPH_GEMM_PF")) : -1;
    // data-tile L2 prefetch distance: off by default (cfg2 Legendre fwd 2.46 ms at 0 vs
    // 2.52 / 2.52 / 2.57 ms at 2 / 4 / 8 k-blocks ahead, profiles/gemm_pf.sh)
    const int pf_dist = pf_env >= 0 ? pf_env : 0;
    // L2 cache hints: 1 evict-first output stores, 2 evict-last table loads (pair kernel).
    // cfg2 round trip 9.33 -> 9.23 ms with both (profiles/r2/gemm_l2hint_sweep.log)
    static const int l2hint = std::getenv("SPH_GEMM_L2HINT") ? std::atoi(std::getenv("SPH_GEMM_L2HINT")) : 3;
    long long* trace = nullptr;
    if (trace_dir) {
        SPH_CUDA(cudaMalloc(&trace, (6 * 512 + 4096) * sizeof(long long)));
        SPH_CUDA(cudaMemsetAsync(trace, 0, (6 * 512 + 4096) * sizeof(long long), st));
    }
    SPH_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mbh, mbl, md, static_cast<const GemmWork*>(tl.d.p),
                                static_cast<int>(tl.n), D,
                                g.store, three ? 1 : 0, trace, dbg, tstore ? 1 : 0,
                                quad ? (quad_rows(g) == 64 ? 3 : quad_rows(g) == 32 ? 2 : 1) : 0, g.d_mode, static_cast<int>(g.d_t),
                                static_cast<int>(g.d_g2), pf_dist, epi, l2hint, (three && g.blo_conv) ? 1 : 0));
    count_launch();
    if (trace) {
        std::vector<long long> h(6 * 512 + 4096);
        SPH_CUDA(cudaStreamSynchronize(st));
        SPH_CUDA(cudaMemcpy(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        cudaFree(trace);
        const std::string path = std::string(trace_dir) + "/gemm_trace_" + g.name + ".txt";
        if (FILE* f = std::fopen(path.c_str(), "w")) {
            for (int j = 0; j < 512; ++j)
                std::fprintf(f, "%d %lld %lld %lld %lld\n", j, h[j], h[512 + j], h[1024 + j], h[1536 + j]);
            std::fclose(f);
        }
        const std::string gpath = std::string(trace_dir) + "/gemm_pairconv_" + g.name + ".txt";
        if (FILE* f = std::fopen(gpath.c_str(), "w")) {  // global-ns conversion stamps, CTA 0 / 1
            for (int j = 0; j < 512; ++j) std::fprintf(f, "%d %lld %lld\n", j, h[2048 + 4096 + j], h[2048 + 4096 + 512 + j]);
            std::fclose(f);
        }
        const std::string tpath = std::string(trace_dir) + "/gemm_tiles_" + g.name + ".txt";
        if (FILE* f = std::fopen(tpath.c_str(), "w")) {
            for (int t = 0; t < 2048; ++t) std::fprintf(f, "%lld %lld\n", h[2048 + 2 * t], h[2048 + 2 * t + 1]);
            std::fclose(f);
        }
    }
}

}  // namespace tc

namespace {
thread_local int t_sm_cap = 0;
}
GemmSmCap::GemmSmCap(int sms) : prev(t_sm_cap) { t_sm_cap = sms; }
GemmSmCap::~GemmSmCap() { t_sm_cap = prev; }
int gemm_sm_cap() { return t_sm_cap; }

void gemm_run_simt(const GroupedGemm& g, const float* A, const float* Bhi, const float* Blo,
                   float* D, cudaStream_t st, const GemmEpi& epi);
void build_simt_tiles(GroupedGemm& g);                                  // gemm_simt.cu

void gemm_run(const GroupedGemm& g, const float* A, float* D, int prec, cudaStream_t st,
              const float* Bhi, const float* Blo, const GemmEpi* epip) {
    const GemmEpi epi = epip ? *epip : GemmEpi{};
    if (g.ntiles == 0) return;
    if (!Bhi) Bhi = g.Bhi.p;
    if (!Blo) Blo = g.Blo.p;
    if (prec == SPH_PREC_FP32_SIMT) {
        gemm_run_simt(g, A, Bhi, Blo, D, st, epi);
        return;
    }
    const bool three = prec == SPH_PREC_3XTF32;
    require(!three || Blo || g.blo_conv, "gemm: 3xTF32 needs the lo table");
    require(!g.blo_conv || g.bn == 192, "gemm: converter-formed B_lo only in the A_lo-in-TMEM bn=192 kernel");
    if (!Blo) Blo = Bhi;  // unused by the kernel when the converter forms B_lo
    const int cl = g.cluster;
    if (g.bn == 192 && g.pair && g.ks == 2)
        tc::launch<192, 2, 2, true, true, 2>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 192 && g.pair)
        tc::launch<192, 4, 2, true, true>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 192 && cl == 1)
        tc::launch<192, 3, 1, true>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 192 && cl == 2)
        tc::launch<192, 3, 2, true>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 192 && cl == 4)
        tc::launch<192, 3, 4, true>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.alo && g.ks == 2 && g.bn == 128 && cl == 1)
        tc::launch<128, 2, 1, true, false, 2>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.alo && g.ks == 2 && g.bn == 128 && cl == 2)
        tc::launch<128, 2, 2, true, false, 2>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.alo && g.ks == 2 && g.bn == 64 && cl == 1)
        tc::launch<64, 3, 1, true, false, 2>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.alo && g.ks == 2 && g.bn == 64 && cl == 2)
        tc::launch<64, 3, 2, true, false, 2>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.alo && g.bn == 128 && cl == 1)
        tc::launch<128, 3, 1, true>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.alo && g.bn == 128 && cl == 2)
        tc::launch<128, 3, 2, true>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.alo && g.bn == 64 && cl == 1)
        tc::launch<64, 4, 1, true>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.alo && g.bn == 64 && cl == 2)
        tc::launch<64, 4, 2, true>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 256 && cl == 1)
        tc::launch<256, 4, 1>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 256 && cl == 2)
        tc::launch<256, 4, 2>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 256 && cl == 4)
        tc::launch<256, 4, 4>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 128 && cl == 1)
        tc::launch<128, 6, 1>(g, A, Bhi, Blo, D, three, st, epi);
    else if (g.bn == 128 && cl == 2)
        tc::launch<128, 6, 2>(g, A, Bhi, Blo, D, three, st, epi);
    else
        fail(SPH_ERR_INVALID_ARGUMENT, "gemm: unsupported N tile");
}

// LPT-ordered tile list for cluster size cl: one entry per (group, n-tile, run of
// cl consecutive M-tiles); ties keep group-major order so concurrently running
// clusters share table tiles in L2.
static void build_tiles(const GroupedGemm& g, int cl, GemmTileList& out) {
    // Groups by cost (see the order note below), and inside a group the N-tiles of
    // one M-run adjacent: concurrently running CTAs then share the data (A) tile in
    // L2 instead of re-reading it from HBM for the second N-tile.
    std::vector<size_t> gorder;
    std::vector<double> gcost(g.groups.size(), 0.0);
    for (size_t gi = 0; gi < g.groups.size(); ++gi) {
        const GemmGroup& gr = g.groups[gi];
        if (gr.M <= 0 || gr.N <= 0 || gr.K <= 0) continue;
        gcost[gi] = static_cast<double>(gr.N) * gr.K;
        gorder.push_back(gi);
    }
    std::stable_sort(gorder.begin(), gorder.end(), [&](size_t a, size_t b) { return gcost[a] > gcost[b]; });
    // Alternate the longest and the shortest remaining groups (SPH_GEMM_ORDER=0: plain
    // decreasing cost), so a CTA's short-K, epilogue-bound tiles sit between long ones whose
    // MMAs hide their epilogues: cfg2 Legendre inverse 2.21 -> 2.11 ms, forward 2.45 -> 2.40
    // (profiles/r2/gemm_order_cmp.log)
    static const int order = std::getenv("SPH_GEMM_ORDER") ? std::atoi(std::getenv("SPH_GEMM_ORDER")) : 1;
    if (order == 1 && gorder.size() > 2) {
        std::vector<size_t> alt;
        alt.reserve(gorder.size());
        for (size_t lo = 0, hi = gorder.size(); lo < hi;) {
            alt.push_back(gorder[lo++]);
            if (lo < hi) alt.push_back(gorder[--hi]);
        }
        gorder.swap(alt);
    }
    std::vector<GemmWork> ts;
    for (size_t gi : gorder) {
        const GemmGroup& gr = g.groups[gi];
        for (int m0 = 0; m0 < gr.M; m0 += tc::BM * cl)
            for (int n0 = 0; n0 < gr.N; n0 += g.bn) {
                GemmWork w{};
                w.a_row = gr.a_row0 + m0;
                w.b_row = gr.b_row0 + n0;
                w.M = gr.M;
                w.m0 = m0;
                w.n0 = n0;
                w.nrem = std::min(g.bn, gr.N - n0);
                w.K = gr.K;
                w.ldd = gr.ldd;
                w.ncols = std::max(w.nrem, std::min(gr.zero_to, n0 + g.bn) - n0);
                w.dg = (g.tma_store || g.d_mode == 1) ? static_cast<int32_t>(gr.d_off / (g.d_rows * g.d_ldd)) : 0;
                w.ag = g.a_quad ? static_cast<int32_t>(gr.a_row0 / g.a_rows_g) : 0;
                w.d_off = gr.d_off;
                ts.push_back(w);
            }
    }
    out.n = static_cast<int64_t>(ts.size());
    out.d.alloc(std::max<size_t>(ts.size(), 1), false);
    if (!ts.empty())
        SPH_CUDA(cudaMemcpy(out.d.p, ts.data(), ts.size() * sizeof(GemmWork), cudaMemcpyHostToDevice));
}

const GemmTileList& GroupedGemm::tiles_for(int cl) const {
    std::lock_guard<std::mutex> lk(*tiles_mu);
    auto& slot = tile_lists[cl];
    if (!slot) {
        slot = std::make_unique<GemmTileList>();
        build_tiles(*this, cl, *slot);
    }
    return *slot;
}

void GroupedGemm::finalize() {
    flops = 0;
    int64_t mtiles = 0;
    for (const GemmGroup& gr : groups) {
        if (gr.M <= 0 || gr.N <= 0 || gr.K <= 0) continue;
        flops += 2.0 * gr.M * static_cast<double>(gr.N) * gr.K;
        mtiles = std::max<int64_t>(mtiles, (gr.M + tc::BM - 1) / tc::BM);
    }
    d_groups.alloc(std::max<size_t>(groups.size(), 1), false);
    if (!groups.empty())
        SPH_CUDA(cudaMemcpy(d_groups.p, groups.data(), groups.size() * sizeof(GemmGroup),
                            cudaMemcpyHostToDevice));
    // table-tile multicast over clusters on neighbouring M-tiles (measured at cfg2,
    // cluster 1 / 2 / 4: Legendre fwd 4.6 / 3.5 / 3.4 ms, inv 4.9 / 4.1 / 3.55 ms)
    // (the pair-mode Legendre GEMMs ignore this; the non-pair GEMMs measured best at 2:
    // cfg4 MLP1 1.36 -> 1.24 ms, MLP2 0.69 -> 0.64 ms, cfg3 DISCO mix 1.445 -> 1.386 ms vs 4)
    if (cluster == 0) cluster = mtiles >= 4 ? 2 : 1;
    if (const char* e = std::getenv("SPH_GEMM_CLUSTER")) {  // test / tuning override
        const int v = std::atoi(e);
        if (v == 1 || v == 2 || v == 4) cluster = v;
    }
    if (alo && bn != 64 && bn != 128) alo = false;
    // two 32-wide atoms per pipeline stage (half the barrier rounds) for the pair and the
    // narrow A_lo-in-TMEM kernels
    if (const char* e = std::getenv("SPH_GEMM_KS")) ks = std::atoi(e) == 2 ? 2 : 1;
    if ((bn == 128 || alo) && cluster > 2) cluster = 2;
    require(!a_quad || (bn == 192 && a_rows_g > 0 && a_kq > 0), "gemm: quad A layout needs the bn=192 kernel");
    // CTA-pair MMA for the BN = 192 (ALO) GEMMs when there are >= 2 M-tiles per group
    pair = bn == 192 && mtiles >= 2;
    if (const char* e = std::getenv("SPH_GEMM_PAIR")) pair = pair && std::atoi(e) != 0;
    // TMA-store epilogue when D is a uniform [group][rows][ldd] array (the Legendre GEMMs)
    tma_store = (bn == 192 || alo || (row_tma && store == STORE_ROW)) && !groups.empty();
    d_rows = 0;
    d_ldd = 0;
    int64_t gmax = 0;
    for (const GemmGroup& gr : groups) {
        if (gr.M <= 0 || gr.N <= 0 || gr.K <= 0) continue;
        const int64_t rows = store == STORE_ROW ? gr.M : gr.N;
        if (d_rows == 0) { d_rows = rows; d_ldd = gr.ldd; }
        if (rows != d_rows || gr.ldd != d_ldd || gr.d_off % (rows * gr.ldd) != 0) tma_store = false;
        if (d_rows > 0) gmax = std::max<int64_t>(gmax, gr.d_off / (d_rows * d_ldd));
    }
    const bool uniform = tma_store;
    if (d_rows == 0 || d_ldd * 4 % 16 != 0) tma_store = false;
    require(d_mode == 0 || (store == STORE_TRANS && bn == 192 && uniform && d_rows > 0),
            "gemm: tiled D layout needs uniform transposed groups");
    if (d_mode == 1 && d_rows > 0) tma_store = true;  // the 4D map has no row-stride constraint
    d_groups3 = gmax + 1;
    if (const char* e = std::getenv("SPH_GEMM_TMA_STORE")) tma_store = tma_store && std::atoi(e) != 0;
    tile_lists.clear();
    ntiles = tiles_for(1).n;
    build_simt_tiles(*this);
}

static inline float rna_tf32(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return x;  // inf/nan untouched
    u += 0x1000u;                                    // round to nearest (ties away)
    u &= 0xffffe000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

void tf32_split_host(const float* x, size_t n, float* hi, float* lo) {
    for (size_t i = 0; i < n; ++i) {
        const float h = rna_tf32(x[i]);
        hi[i] = h;
        lo[i] = x[i] - h;
    }
}

}  // namespace sph
