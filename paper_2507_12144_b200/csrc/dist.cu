// Domain-decomposed SHT (forward + inverse) and DISCO over NCCL: the paper's Algorithms
// 1-2 (distsim.hpp:404-547) on real GPUs, one process per GPU.  The host layout logic
// (who owns what, who sends what) is dist_layout.hpp; this file owns the communicators,
// the pack / unpack kernels and the stage order.  Every collective is a grouped
// ncclSend/ncclRecv all-to-all (canonical uneven splits) or ncclReduceScatter on the
// caller's stream, so a call is stream-ordered like every other library call.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "capi_util.cuh"
#include "dist_layout.hpp"
#include "tile_rows.cuh"

namespace sph {

// NCCL is bound at run time, on the first communicator: the copy already in the process
// (e.g. the one PyTorch links) when there is one, else libnccl.so.2 from the loader path
// (SPH_NCCL_LIB overrides).  libsphgpu.so itself has no NCCL dependency, so loading it
// never pins an NCCL version that a later import would conflict with.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        const char* env = std::getenv("SPH_NCCL_LIB");
        void* h = env ? dlopen(env, RTLD_NOW | RTLD_GLOBAL) : dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h && !env) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("cannot load NCCL: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && err.empty()) err = std::string("NCCL symbol missing: ") + name;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommSplit, "ncclCommSplit");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.ReduceScatter, "ncclReduceScatter");
        sym(api.GetErrorString, "ncclGetErrorString");
    });
    if (!err.empty()) fail(SPH_ERR_NCCL, err);
    return api;
}

inline void nccl_check(ncclResult_t r, const char* what, const char* file, int line) {
    if (r != ncclSuccess)
        fail(SPH_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r) + " (" + file + ":" +
                               std::to_string(line) + ")");
}
#define SPH_NCCL(x) ::sph::nccl_check((x), #x, __FILE__, __LINE__)

// TrafficLog of the reference (distsim.hpp:120-150): bytes are summed over all ranks
// (every rank knows every rank's payload sizes from the layout, so no communication).
struct Traffic {
    struct Rec {
        std::string op, axis, coll;
        int64_t bytes = 0, calls = 0;
    };
    std::vector<Rec> recs;
    void record(const std::string& op, const std::string& axis, const std::string& coll, int64_t bytes) {
        for (auto& r : recs)
            if (r.op == op && r.axis == axis && r.coll == coll) {
                r.bytes += bytes;
                r.calls += 1;
                return;
            }
        recs.push_back({op, axis, coll, bytes, 1});
    }
    std::string csv() const {
        std::string out = "operation,axis,collective,bytes,calls\n";
        for (const auto& r : recs)
            out += r.op + "," + r.axis + "," + r.coll + "," + std::to_string(r.bytes) + "," + std::to_string(r.calls) + "\n";
        return out;
    }
};

}  // namespace sph

// The rank's communicator hierarchy (distsim.hpp:45-98, 160-163): the world, the
// (polar x azimuth) plane of its (batch, ensemble) coordinate, and its azimuth group,
// all split from the world communicator with ncclCommSplit.
struct sph_comm_s {
    int device = 0;
    sph::CommGridSpec grid;
    int64_t rank = 0;
    std::array<int64_t, 4> coords{};
    int64_t plane_rank = 0, plane_size = 1;
    int nccl_ctas = 32;  // maxCTAs of the plane communicator (SPH_NCCL_MAX_CTAS)
    ncclComm_t world = nullptr, plane = nullptr, az = nullptr;
    std::mutex mu;
    sph::Traffic log;
    ~sph_comm_s() {
        for (ncclComm_t c : {az, plane, world})
            if (c) sph::nccl().CommDestroy(c);
    }
};

namespace sph {
namespace {

// ------------------------------------------------------------------------- kernels
struct DBox {
    int64_t src_off, dst_off, n0, n1, n2, s0, s1, d0, d1, row0;
    int32_t vec4, pad;
};

// One warp per row (n2 contiguous floats) of the flattened box list; float4 when every
// offset, stride and width of the box is a multiple of 4.
__global__ void __launch_bounds__(256) box_copy_kernel(const DBox* __restrict__ bx, int nbox, int64_t rows,
                                                       const float* __restrict__ src, float* __restrict__ dst) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (r >= rows) return;
    int b = 0;
    while (b + 1 < nbox && bx[b + 1].row0 <= r) ++b;
    const DBox& B = bx[b];
    const int64_t rr = r - B.row0, a = rr / B.n1, c = rr - a * B.n1;
    const float* s = src + B.src_off + a * B.s0 + c * B.s1;
    float* d = dst + B.dst_off + a * B.d0 + c * B.d1;
    const int lane = threadIdx.x & 31;
    if (B.vec4) {
        const float4* s4 = reinterpret_cast<const float4*>(s);
        float4* d4 = reinterpret_cast<float4*>(d);
        for (int64_t k = lane; k < B.n2 / 4; k += 32) d4[k] = __ldg(s4 + k);
    } else {
        for (int64_t k = lane; k < B.n2; k += 32) d[k] = __ldg(s + k);
    }
}

// Coefficient payload index (complex units) of (field f, degree l, order m), m <= l:
//   off[p] + f * tri[p] + rowoff[robase[p] + l - l0(i)] + m - m0(j),  p = i * nw + j
// with (i, l - l0) = lmap[l], (j, m - m0) = mmap[m]  (dist_layout.hpp, ShtLayout).
// The host flattens everything but the field term into per-(degree, order block) tables,
//   b0[l * nw + j] = off[p] + rowoff[robase[p] + l - l0(i)] - m0(j),  tr[l * nw + j] = tri[p]
// so a tile stages rowbase(f, l, j) = b0 + f * tr with two independent loads (the chained
// lmap -> off / tri / robase -> rowoff lookups were a 4-deep dependent-load chain per CTA).
struct PayloadMap {
    const int2* mmap;
    const int64_t* b0;
    const int64_t* tr;
    int nw;
};
constexpr int kMaxNw = 16;  // azimuth ranks a staged tile supports (>= every B200 box)

// stage base[ll][j] = rowbase(f, lt + ll, j) for the tile's degrees and the order blocks
// j its 32 orders touch (jlo .. jlo + nj - 1)
__device__ __forceinline__ void stage_rowbase(int64_t* base, const PayloadMap& pm, int64_t f, int lt, int nl,
                                              int lmax, int mt, int mmax, int& jlo, int& nj) {
    const int mlast = min(mt + 31, mmax - 1);
    jlo = pm.mmap[mt].x;
    nj = pm.mmap[mlast].x - jlo + 1;
    for (int e = threadIdx.x; e < nl * nj; e += blockDim.x) {
        const int ll = e / nj, jj = e - ll * nj;
        const int l = lt + ll;
        if (l < lmax) {
            const int64_t t = static_cast<int64_t>(l) * pm.nw + jlo + jj;
            base[ll * kMaxNw + jj] = __ldg(pm.b0 + t) + f * __ldg(pm.tr + t);
        }
    }
}

// forward B pack: the local SHT's C_int [(m*2+p)][2F][Lp] (l = m + p + 2 lp) -> triangular
// payloads of every destination block.  CTA (32 orders, 64 degrees, field f): C_int rows
// read as 32-lane lp runs, payload written in order runs (indexing: tile_rows.cuh).
__global__ void __launch_bounds__(256) cint_pack_kernel(const float* __restrict__ cint, int64_t F, int lmax, int mmax,
                                                        int Lp, PayloadMap pm, float2* __restrict__ payload) {
    constexpr int DL = 64, RPW = 128 / 8;
    __shared__ float tre[DL][33], tim[DL][33];
    __shared__ int64_t base[DL * kMaxNw];
    const int mt = blockIdx.x * 32, lt = blockIdx.y * DL;
    if (mt > lt + DL - 1) return;  // tile entirely above the diagonal (m > l)
    const int64_t f = blockIdx.z;
    int jlo, nj;
    stage_rowbase(base, pm, f, lt, DL, lmax, mt, mmax, jlo, nj);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {  // a warp's 16 rows: all loads issued before any shared-memory store
        const int p = (warp >> 1) & 1, ri = warp & 1;
        float (*T)[33] = ri ? tim : tre;
        const int64_t gstep = 8 * F * Lp;  // 4 groups (m += 2)
        const int mw = mt + (warp >> 2);
        const float* rp = cint + ((static_cast<int64_t>(mw) * 2 + p) * 2 * F + 2 * f + ri) * Lp + lane;
        float v[RPW];
        int sr[RPW];
        int d = lt - mw - p;  // TileRow offset, -2 per row
#pragma unroll
        for (int i = 0; i < RPW; ++i, d -= 2, rp += gstep) {
            const TileRow tr(d);
            const int lp = tr.lp0 + lane, dl = tr.off0 + 2 * lane;
            const bool ok = mw + 2 * i < mmax && dl < DL && lp < Lp && lt + dl < lmax;
            v[i] = ok ? __ldg(rp + tr.lp0) : 0.f;
            sr[i] = ok ? tr.s0 + lane : -1;
        }
#pragma unroll
        for (int i = 0; i < RPW; ++i)
            if (sr[i] >= 0) T[sr[i]][(warp >> 2) + 2 * i] = v[i];
    }
    __syncthreads();
    const int m = mt + lane;  // this thread's order
    if (m >= mmax) return;
    const int jme = pm.mmap[m].x - jlo;
#pragma unroll
    for (int i = 0; i < DL / 8; ++i) {
        const int dl = warp + 8 * i, l = lt + dl;
        if (l >= lmax || m > l) continue;
        const int sr = (warp & 1) * (DL / 2) + (warp >> 1) + 4 * i;
        payload[base[dl * kMaxNw + jme] + m] = make_float2(tre[sr][lane], tim[sr][lane]);
    }
}

// inverse A^-1 unpack: triangular payloads of every source block -> C_int of the local
// fields.  CTA (32 orders, 64 degrees, field f): the tile's payload entries loaded once in
// order runs, each (order, parity, re/im) C_int row's 32 lp of the tile written as one
// run; degree tiles run to lmax + 63 so every lp the inverse GEMM reads (L(m, p) rounded
// to its 32-wide k-block) is written, zeros beyond lmax.
template <int FPC>
__global__ void __launch_bounds__(256) cint_unpack_kernel(const float2* __restrict__ payload, int64_t F, int lmax,
                                                          int mmax, int Lp, PayloadMap pm, float* __restrict__ cint) {
    constexpr int DL = 64, RPW = 128 / 8, EPT = DL * 32 / 256;
    __shared__ float tre[FPC][DL][33], tim[FPC][DL][33];
    __shared__ int64_t base[DL * kMaxNw];
    __shared__ int32_t trs[FPC > 1 ? DL * kMaxNw : 1];  // per-field payload stride (field q: + q * trs)
    const int mt = blockIdx.x * 32, lt = blockIdx.y * DL;
    const int64_t f = static_cast<int64_t>(blockIdx.z) * FPC;
    const int nf = static_cast<int>(min(static_cast<int64_t>(FPC), F - f));
    int jlo, nj;
    stage_rowbase(base, pm, f, lt, DL, lmax, mt, mmax, jlo, nj);
    if (FPC > 1)
        for (int e = threadIdx.x; e < DL * nj; e += blockDim.x) {
            const int ll = e / nj, jj = e - ll * nj;
            if (lt + ll < lmax) trs[ll * kMaxNw + jj] = static_cast<int32_t>(__ldg(pm.tr + static_cast<int64_t>(lt + ll) * pm.nw + jlo + jj));
        }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {  // element i: degree lt + warp + 8 i, order mt + lane; all loads before the stores
        const int m = mt + lane;
        const int jme = m < mmax ? pm.mmap[m].x - jlo : 0;
        float2 v[FPC][EPT];
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int dl = warp + 8 * i, l = lt + dl;
            const bool ok = l < lmax && m < mmax && m <= l;
            const int64_t at = ok ? base[dl * kMaxNw + jme] + m : 0;
            const int64_t fs = FPC > 1 && ok ? trs[dl * kMaxNw + jme] : 0;
#pragma unroll
            for (int q = 0; q < FPC; ++q)
                v[q][i] = ok && q < nf ? __ldg(payload + at + q * fs) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < FPC; ++q)
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int sr = (warp & 1) * (DL / 2) + (warp >> 1) + 4 * i;
                tre[q][sr][lane] = v[q][i].x;
                tim[q][sr][lane] = v[q][i].y;
            }
    }
    __syncthreads();
    const int p = (warp >> 1) & 1, ri = warp & 1;
    const int64_t gstep = 8 * F * Lp;  // 4 groups (m += 2)
    const int mw = mt + (warp >> 2);
    float* rp = cint + ((static_cast<int64_t>(mw) * 2 + p) * 2 * F + 2 * f + ri) * Lp + lane;
    int d = lt - mw - p;               // TileRow offset, -2 per row
    int lmp = (lmax - mw + 1 - p) >> 1;  // L(m, p) while m < lmax (<= 0 after), -1 per row
#pragma unroll
    for (int i = 0; i < RPW; ++i, d -= 2, --lmp, rp += gstep) {
        if (mw + 2 * i >= mmax) break;
        const TileRow tr(d);
        const int lp = tr.lp0 + lane, dl = tr.off0 + 2 * lane;
        const int lim = min(Lp, (max(lmp, 0) + 31) & ~31);
        if (dl < DL && lp < lim) {
            const bool in = lt + dl < lmax;
#pragma unroll
            for (int q = 0; q < FPC; ++q)
                if (q < nf) rp[tr.lp0 + q * 2 * Lp] = in ? (ri ? tim : tre)[q][tr.s0 + lane][(warp >> 2) + 2 * i] : 0.f;
        }
    }
}

// forward B unpack / inverse A^-1 pack: the rank's own dense block [C][ln][mn] complex
// (reference unshard layout, zeros above the diagonal) <-> [C][tri] channel-major payload.
// One CTA per (channel, degree) row; the row's payload run starts at c*tri + rowoff[k].
template <bool TO_BLOCK>
__global__ void __launch_bounds__(256) block_tri_kernel(float2* __restrict__ block, float2* __restrict__ payload,
                                                        int ln, int mn, int l0, int m0,
                                                        const int64_t* __restrict__ rowoff, int64_t tri) {
    const int k = blockIdx.x;
    const int64_t c = blockIdx.y;
    const int nvalid = min(mn, max(0, l0 + k + 1 - m0));  // orders m0 .. l0+k of this row
    float2* brow = block + (c * ln + k) * mn;
    float2* prow = payload + c * tri + rowoff[k];
    for (int jm = threadIdx.x; jm < mn; jm += blockDim.x) {
        if (TO_BLOCK) brow[jm] = jm < nvalid ? prow[jm] : make_float2(0.f, 0.f);
        else if (jm < nvalid) prow[jm] = brow[jm];
    }
}

// ---------------------------------------------------------------- host helpers
struct BoxList {
    DevBuf<DBox> d;
    int n = 0;
    int64_t rows = 0, floats = 0;
    void set(const std::vector<Box>& bs) {
        std::vector<DBox> h;
        rows = floats = 0;
        for (const Box& b : bs) {
            if (b.n0 * b.n1 * b.n2 == 0) continue;
            DBox x{b.src_off, b.dst_off, b.n0, b.n1, b.n2, b.s0, b.s1, b.d0, b.d1, rows, 0, 0};
            x.vec4 = (b.src_off % 4 == 0 && b.dst_off % 4 == 0 && b.n2 % 4 == 0 && b.s0 % 4 == 0 && b.s1 % 4 == 0 &&
                      b.d0 % 4 == 0 && b.d1 % 4 == 0);
            rows += b.n0 * b.n1;
            floats += b.n0 * b.n1 * b.n2;
            h.push_back(x);
        }
        n = static_cast<int>(h.size());
        d.alloc(h.size(), false);
        if (!h.empty()) SPH_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(DBox), cudaMemcpyHostToDevice));
    }
    // src/dst must be 16-byte aligned for the float4 boxes (workspace carve-outs are)
    void run(const float* src, float* dst, cudaStream_t st, const char* name) const {
        if (!rows) return;
        ProfScope prof(name, st, 8.0 * static_cast<double>(floats));
        box_copy_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(d.p, n, rows, src, dst);
        SPH_LAUNCH_CHECK();
        count_launch();
    }
};

template <class T>
void upload_vec(DevBuf<T>& d, const std::vector<T>& h) {
    d.alloc(h.size(), false);
    if (!h.empty()) SPH_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

// grouped point-to-point all-to-all over `comm` (plane ranks); the self block is a
// device-to-device copy
void alltoallv(ncclComm_t comm, int64_t me, const Exchange& x, const float* send, float* recv, cudaStream_t st) {
    const int64_t P = static_cast<int64_t>(x.send_cnt.size());
    if (x.send_cnt[me]) {
        require(x.send_cnt[me] == x.recv_cnt[me], "all_to_all: self block size mismatch");
        if (send + x.send_off[me] != recv + x.recv_off[me])
            SPH_CUDA(cudaMemcpyAsync(recv + x.recv_off[me], send + x.send_off[me], 4 * x.send_cnt[me],
                                     cudaMemcpyDeviceToDevice, st));
    }
    if (P == 1) return;
    SPH_NCCL(sph::nccl().GroupStart());
    for (int64_t p = 0; p < P; ++p) {
        if (p == me) continue;
        if (x.send_cnt[p])
            SPH_NCCL(sph::nccl().Send(send + x.send_off[p], static_cast<size_t>(x.send_cnt[p]), ncclFloat, static_cast<int>(p),
                              comm, st));
        if (x.recv_cnt[p])
            SPH_NCCL(sph::nccl().Recv(recv + x.recv_off[p], static_cast<size_t>(x.recv_cnt[p]), ncclFloat, static_cast<int>(p),
                              comm, st));
    }
    SPH_NCCL(sph::nccl().GroupEnd());
}

// world-summed remote bytes of one exchange (the reference TrafficLog accounting)
template <class XFn>
int64_t world_bytes(int64_t P, int64_t planes, XFn xfn) {
    int64_t b = 0;
    for (int64_t q = 0; q < P; ++q) b += 4 * xfn(q).remote_send(q);
    return b * planes;
}

struct Carve {  // 256-byte aligned sub-buffers of one workspace
    int64_t off = 0;
    int64_t take(int64_t bytes) {
        const int64_t o = off;
        off += static_cast<int64_t>(round_up(static_cast<size_t>(std::max<int64_t>(bytes, 0)), 256));
        return o;
    }
};

}  // namespace
}  // namespace sph

// ------------------------------------------------------------------ distributed SHT
namespace sph {
namespace {
// One channel chunk of the distributed SHT: an independent Alg. 1 problem on channels
// [c_begin, c_begin + C_k) (its own canonical channel slices, exchanges and boxes).
struct ShtChunk {
    ShtLayout lay;
    int64_t c_begin = 0;
    Exchange xa, xb, xia, xib;
    BoxList fwd_unpack, inv_pack;
    // nw == 1: every stage block holds whole rings, so the ring transforms address the
    // stage buffers in place through per-latitude tables (fft.cuh RingRows: roff, then
    // fstr, nlat each) and the unpack / pack box copies are skipped
    bool direct = false;
    DevBuf<int64_t> rows_a, rows_b;
    RingRows ring_a() const { return {rows_a.p, rows_a.p ? rows_a.p + rows_a.n / 2 : nullptr}; }
    RingRows ring_b() const { return {rows_b.p, rows_b.p ? rows_b.p + rows_b.n / 2 : nullptr}; }
    DevBuf<int64_t> b0_b, b0_ia;  // flattened payload row bases per (degree, order block) (PayloadMap)
    std::vector<int64_t> off_b_h, off_ia_h;  // payload offsets per block (complex units)
    int64_t bytes_fa = 0, bytes_fb = 0, bytes_ia = 0, bytes_ib = 0;
};

struct Events {
    std::vector<cudaEvent_t> ev;
    cudaEvent_t make() {
        cudaEvent_t e;
        SPH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev.push_back(e);
        return e;
    }
    ~Events() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
};
}  // namespace
}  // namespace sph

// Channel chunks are software-pipelined over two streams: the caller's stream runs the
// compute (unpack, fused SHT, pack) and an internal stream issues every NCCL exchange, so
// chunk k+1's inbound all-to-all and chunk k-1's outbound one run while chunk k computes.
// During the overlapped region the persistent GEMM leaves SPH_NCCL_MAX_CTAS SMs to the
// NCCL kernels (GemmSmCap; the plane communicator is split with that maxCTAs).  Buffers
// that cross streams are double-buffered (set k % 2) and guarded by events.
struct sph_dist_sht_plan_s {
    sph_comm comm = nullptr;
    sph::ShtPlan* sht = nullptr;
    sph::ShtLayout lay;  // the whole problem (ranges reported to the caller)
    int64_t q = 0, i = 0, j = 0;
    std::vector<std::unique_ptr<sph::ShtChunk>> chunks;
    sph::DevBuf<int2> mmap;
    sph::DevBuf<int64_t> tr, rowoff_me;
    int64_t tri_me = 0;
    // workspace carve (bytes): stage / pay / mine are double-buffered
    int64_t o_stage[2] = {0, 0}, o_pay[2] = {0, 0}, o_mine[2] = {0, 0};
    int64_t o_full = 0, o_cint = 0, o_shtws = 0, total = 0;
    cudaStream_t cs = nullptr;
    sph::Events evs;
    cudaEvent_t e_start = nullptr, e_end = nullptr;
    cudaEvent_t eA[2], eUA[2], eP[2], eB[2], eP1[2], eA1[2], eUC[2], eP2[2], eB2[2];
    int sm_cap = 0;
    std::mutex mu, call_mu;
    sph::DevBuf<uint8_t> own_ws;

    ~sph_dist_sht_plan_s() {
        if (cs) {
            cudaStreamSynchronize(cs);
            cudaStreamDestroy(cs);
        }
    }

    void create(sph_comm c, sph::ShtPlan* p, int64_t C) {
        using namespace sph;
        comm = c;
        sht = p;
        const int64_t nh = c->grid.sizes[2], nw = c->grid.sizes[3];
        lay = ShtLayout(nh, nw, p->nlat, p->nlon, p->lmax, p->mmax, C);
        require(nw <= kMaxNw, "dist_sht: at most 16 azimuth ranks");
        require(C <= 65535 && p->lmax <= 65535, "dist_sht: too many channels for one call");
        q = c->plane_rank;
        i = lay.pi(q);
        j = lay.pj(q);
        DeviceGuard dg(p->device);
        // channel chunks: >= one channel per rank and chunk, SPH_DIST_CHUNKS (default 4)
        static const int64_t want = [] {
            const char* e = std::getenv("SPH_DIST_CHUNKS");
            return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t{2};
        }();
        const int64_t nchunk = lay.P == 1 ? 1 : std::max<int64_t>(1, std::min(want, C / lay.P));
        const std::vector<int64_t> csplit = canonical_split(C, nchunk);
        const int64_t planes = c->grid.sizes[0] * c->grid.sizes[1];
        const int64_t HW = p->nlat * p->nlon;
        int64_t m_stage = 0, m_full = 0, m_cint = 0, m_ws = 0, m_pay = 0, m_mine = 0;
        for (int64_t k = 0; k < nchunk; ++k) {
            auto ch = std::make_unique<ShtChunk>();
            ch->lay = ShtLayout(nh, nw, p->nlat, p->nlon, p->lmax, p->mmax, csplit[k]);
            ch->c_begin = split_offset(csplit, k);
            const ShtLayout& L = ch->lay;
            ch->xa = L.fwd_fields(q);
            ch->xb = L.fwd_coeffs(q);
            ch->xia = L.inv_coeffs(q);
            ch->xib = L.inv_fields(q);
            ch->fwd_unpack.set(L.fwd_unpack(q));
            ch->inv_pack.set(L.inv_pack(q));
            ch->direct = nw == 1 && L.cq(q) > 0 && !std::getenv("SPH_DIST_BOXCOPY");
            if (ch->direct) {
                // ring rows of the stage blocks: fields side offset h * nlon, stage side
                // (block offset + c * row stride), per-field stride of the block
                const int64_t nlat = p->nlat, nlon = p->nlon;
                auto tables = [&](const std::vector<Box>& bs, bool fields_is_dst) {
                    std::vector<int64_t> t(2 * nlat, -1);
                    for (const Box& b : bs) {
                        const int64_t foff = fields_is_dst ? b.dst_off : b.src_off;
                        const int64_t soff = fields_is_dst ? b.src_off : b.dst_off;
                        const int64_t fs0 = fields_is_dst ? b.d0 : b.s0, fs1 = fields_is_dst ? b.d1 : b.s1;
                        const int64_t ss0 = fields_is_dst ? b.s0 : b.d0, ss1 = fields_is_dst ? b.s1 : b.d1;
                        require(b.n2 == nlon && foff % nlon == 0 && fs0 == nlat * nlon && fs1 == nlon,
                                "dist_sht: stage block is not whole rings");
                        for (int64_t c = 0; c < b.n1; ++c) {
                            t[foff / nlon + c] = soff + c * ss1;
                            t[nlat + foff / nlon + c] = ss0;
                        }
                    }
                    for (int64_t h = 0; h < nlat; ++h) require(t[h] >= 0, "dist_sht: stage rows do not cover the grid");
                    return t;
                };
                upload_vec(ch->rows_a, tables(L.fwd_unpack(q), true));
                upload_vec(ch->rows_b, tables(L.inv_pack(q), false));
            }
            std::vector<int64_t> ob(L.P), oia(L.P);
            for (int64_t s2 = 0; s2 < L.P; ++s2) {
                ob[s2] = ch->xb.send_off[s2] / 2;
                oia[s2] = ch->xia.recv_off[s2] / 2;
            }
            ch->off_b_h = ob;
            ch->off_ia_h = oia;
            ch->bytes_fa = world_bytes(L.P, planes, [&](int64_t r) { return L.fwd_fields(r); });
            ch->bytes_fb = world_bytes(L.P, planes, [&](int64_t r) { return L.fwd_coeffs(r); });
            ch->bytes_ia = world_bytes(L.P, planes, [&](int64_t r) { return L.inv_coeffs(r); });
            ch->bytes_ib = world_bytes(L.P, planes, [&](int64_t r) { return L.inv_fields(r); });
            const int64_t cq = L.cq(q);
            m_stage = std::max({m_stage, ch->xa.recv_total(), ch->xib.send_total()});
            m_full = std::max(m_full, cq * HW);
            m_cint = std::max(m_cint, p->cint_elems(cq));
            m_ws = std::max(m_ws, p->workspace_bytes(cq));
            m_pay = std::max({m_pay, ch->xb.send_total(), ch->xia.recv_total()});
            m_mine = std::max({m_mine, ch->xb.recv_total(), ch->xia.send_total()});
            chunks.push_back(std::move(ch));
        }
        std::vector<int2> mm(p->mmax);
        for (int64_t b = 0; b < nw; ++b)
            for (int64_t k = 0; k < lay.mp[b]; ++k) mm[lay.m0(b) + k] = make_int2(static_cast<int>(b), static_cast<int>(k));
        upload_vec(mmap, mm);
        // PayloadMap tables: tr[l][j] = tri of block (i(l), j); the chunk's b0[l][j] adds its
        // block offsets (rowoff of block p at degree l, minus the block's first order)
        std::vector<std::vector<int64_t>> rof(lay.P);
        for (int64_t s2 = 0; s2 < lay.P; ++s2) rof[s2] = lay.rowoff(s2);
        tri_me = rof[q].back();
        std::vector<int64_t> trt(p->lmax * nw), rel(p->lmax * nw);
        std::vector<int64_t> pof(p->lmax * nw);
        for (int64_t a = 0; a < nh; ++a)
            for (int64_t k = 0; k < lay.lp[a]; ++k)
                for (int64_t b = 0; b < nw; ++b) {
                    const int64_t t = (lay.l0(a) + k) * nw + b, s2 = a * nw + b;
                    trt[t] = rof[s2].back();
                    rel[t] = rof[s2][k] - lay.m0(b);
                    pof[t] = s2;
                }
        upload_vec(tr, trt);
        for (auto& chp : chunks) {
            std::vector<int64_t> bb(trt.size()), bi(trt.size());
            for (size_t t = 0; t < trt.size(); ++t) {
                bb[t] = chp->off_b_h[pof[t]] + rel[t];
                bi[t] = chp->off_ia_h[pof[t]] + rel[t];
            }
            upload_vec(chp->b0_b, bb);
            upload_vec(chp->b0_ia, bi);
        }
        upload_vec(rowoff_me, rof[q]);
        Carve cv;
        for (int b = 0; b < 2; ++b) o_stage[b] = cv.take(4 * m_stage);
        o_full = cv.take(4 * m_full);
        o_cint = cv.take(4 * m_cint);
        o_shtws = cv.take(m_ws);
        for (int b = 0; b < 2; ++b) o_pay[b] = cv.take(4 * m_pay);
        for (int b = 0; b < 2; ++b) o_mine[b] = cv.take(4 * m_mine);
        total = cv.off;
        if (lay.P > 1) {
            int lo = 0, hi = 0;
            SPH_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            SPH_CUDA(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, hi));
            e_start = evs.make();
            e_end = evs.make();
            for (int b = 0; b < 2; ++b) {
                eA[b] = evs.make();
                eUA[b] = evs.make();
                eP[b] = evs.make();
                eB[b] = evs.make();
                eP1[b] = evs.make();
                eA1[b] = evs.make();
                eUC[b] = evs.make();
                eP2[b] = evs.make();
                eB2[b] = evs.make();
            }
            if (chunks.size() > 1) sm_cap = std::max(16, num_sms() - c->nccl_ctas);
        }
    }
    uint8_t* ws_base(void* ws) {
        if (ws) return static_cast<uint8_t*>(ws);
        std::lock_guard<std::mutex> lk(mu);
        if (own_ws.n < static_cast<size_t>(total)) own_ws.alloc(total, true);
        return own_ws.p;
    }
    sph::PayloadMap pmap(const sph::DevBuf<int64_t>& b0) const {
        return {mmap.p, b0.p, tr.p, static_cast<int>(lay.nw)};
    }
    void log(const char* op, int64_t bytes) {
        std::lock_guard<std::mutex> lk(comm->mu);
        comm->log.record(op, "polar+azimuth", "all_to_all", bytes);
    }
    template <class T>
    static T* at(uint8_t* w, int64_t off) {
        return reinterpret_cast<T*>(w + off);
    }
    void wait(cudaStream_t s, cudaEvent_t e) { SPH_CUDA(cudaStreamWaitEvent(s, e, 0)); }
    void rec(cudaEvent_t e, cudaStream_t s) { SPH_CUDA(cudaEventRecord(e, s)); }

    // x [C][H_i][W_j] -> coeffs [C][L_i][M_j] complex64 (dense, zeros above the diagonal)
    void forward(const float* x, float* out, void* ws, cudaStream_t st) {
        using namespace sph;
        DeviceGuard dg(sht->device);
        require_on_device(x, sht->device, "dist_sht_forward");
        require_on_device(out, sht->device, "dist_sht_forward");
        if (lay.P == 1) {
            sht->forward(x, lay.C, out, SPH_LAYOUT_DENSE_LM, nullptr, st);
            log("dist_sht", 0);
            log("dist_sht", 0);
            return;
        }
        std::lock_guard<std::mutex> call(call_mu);  // the plan's streams / events serve one call at a time
        uint8_t* w = ws_base(ws);
        GemmSmCap cap(sm_cap);
        const int64_t n = static_cast<int64_t>(chunks.size());
        const int64_t fblk = lay.field_block(q), cblk = 2 * lay.lp[i] * lay.mp[j];
        rec(e_start, st);
        wait(cs, e_start);
        int64_t bytes_a = 0, bytes_b = 0;  // one TrafficLog record per exchange of the call
        auto issue_a = [&](int64_t k) {  // inbound exchange of chunk k on the comm stream
            const ShtChunk& ch = *chunks[k];
            const int b = k & 1;
            if (k >= 2) wait(cs, eUA[b]);  // stage[b] consumed by chunk k-2's unpack
            alltoallv(comm->plane, q, ch.xa, x + ch.c_begin * fblk, at<float>(w, o_stage[b]), cs);
            rec(eA[b], cs);
            bytes_a += ch.bytes_fa;
        };
        auto unpack_b = [&](int64_t k) {  // chunk k's received triangles -> its output rows
            const ShtChunk& ch = *chunks[k];
            const int b = k & 1;
            wait(st, eB[b]);
            const int64_t C = ch.lay.C;
            if (C * lay.lp[i] * lay.mp[j]) {
                ProfScope prof("dist_unpack_tri", st, 8.0 * C * lay.lp[i] * lay.mp[j] + 4.0 * ch.xb.recv_total());
                block_tri_kernel<true><<<dim3(static_cast<unsigned>(lay.lp[i]), static_cast<unsigned>(C)),
                                         lay.mp[j] > 128 ? 256 : 128, 0, st>>>(
                    reinterpret_cast<float2*>(out + ch.c_begin * cblk), at<float2>(w, o_mine[b]),
                    static_cast<int>(lay.lp[i]), static_cast<int>(lay.mp[j]), static_cast<int>(lay.l0(i)),
                    static_cast<int>(lay.m0(j)), rowoff_me.p, tri_me);
                SPH_LAUNCH_CHECK();
                count_launch();
            }
        };
        issue_a(0);
        for (int64_t k = 0; k < n; ++k) {
            const ShtChunk& ch = *chunks[k];
            const int b = k & 1;
            const int64_t cq = ch.lay.cq(q);
            if (k + 1 < n) issue_a(k + 1);
            // compute of chunk k on the caller's stream
            wait(st, eA[b]);
            if (!ch.direct) {
                ch.fwd_unpack.run(at<float>(w, o_stage[b]), at<float>(w, o_full), st, "dist_unpack_fields");
                rec(eUA[b], st);
            }
            if (cq > 0) {
                if (ch.direct) {  // the fold reads the received blocks in place
                    sht->forward(at<float>(w, o_stage[b]), cq, at<float>(w, o_cint), SPH_LAYOUT_INTERNAL, w + o_shtws,
                                 st, ch.ring_a());
                    rec(eUA[b], st);
                } else {
                    sht->forward(at<float>(w, o_full), cq, at<float>(w, o_cint), SPH_LAYOUT_INTERNAL, w + o_shtws, st);
                }
                ProfScope prof("dist_pack_cint", st, 4.0 * sht->cint_elems(cq) + 4.0 * ch.xb.send_total());
                constexpr int LT = 64;
                dim3 g(static_cast<unsigned>((lay.mmax + 31) / 32), static_cast<unsigned>((lay.lmax + LT - 1) / LT),
                       static_cast<unsigned>(cq));
                cint_pack_kernel<<<g, 256, 0, st>>>(at<float>(w, o_cint), cq, static_cast<int>(lay.lmax),
                                                        static_cast<int>(lay.mmax), sht->Lp, pmap(ch.b0_b),
                                                        at<float2>(w, o_pay[b]));
                SPH_LAUNCH_CHECK();
                count_launch();
            }
            rec(eP[b], st);
            if (k >= 1) unpack_b(k - 1);  // the previous chunk's outbound exchange has had chunk k's compute to land
            // outbound exchange of chunk k (mine[b] was last read by chunk k-2's unpack, which
            // the caller's stream ran before eP[b])
            wait(cs, eP[b]);
            alltoallv(comm->plane, q, ch.xb, at<float>(w, o_pay[b]), at<float>(w, o_mine[b]), cs);
            rec(eB[b], cs);
            bytes_b += ch.bytes_fb;
        }
        unpack_b(n - 1);
        rec(e_end, cs);
        wait(st, e_end);
        log("dist_sht", bytes_a);
        log("dist_sht", bytes_b);
    }

    // coeffs [C][L_i][M_j] complex64 -> y [C][H_i][W_j]  (mirror of forward)
    void inverse(const float* in, float* y, void* ws, cudaStream_t st) {
        using namespace sph;
        DeviceGuard dg(sht->device);
        require_on_device(in, sht->device, "dist_sht_inverse");
        require_on_device(y, sht->device, "dist_sht_inverse");
        if (lay.P == 1) {
            sht->inverse(in, lay.C, SPH_LAYOUT_DENSE_LM, y, nullptr, st);
            log("dist_isht", 0);
            log("dist_isht", 0);
            return;
        }
        std::lock_guard<std::mutex> call(call_mu);
        uint8_t* w = ws_base(ws);
        GemmSmCap cap(sm_cap);
        const int64_t n = static_cast<int64_t>(chunks.size());
        const int64_t fblk = lay.field_block(q), cblk = 2 * lay.lp[i] * lay.mp[j];
        rec(e_start, st);
        wait(cs, e_start);
        int64_t bytes_a = 0, bytes_b = 0;
        auto pack_tri = [&](int64_t k) {  // chunk k's rows of the own block -> [C_k][tri] (caller's stream)
            const ShtChunk& ch = *chunks[k];
            const int b = k & 1;
            const int64_t C = ch.lay.C;
            if (C * lay.lp[i] * lay.mp[j]) {
                ProfScope prof("dist_pack_tri", st, 8.0 * C * lay.lp[i] * lay.mp[j] + 4.0 * ch.xia.send_total());
                block_tri_kernel<false><<<dim3(static_cast<unsigned>(lay.lp[i]), static_cast<unsigned>(C)),
                                          lay.mp[j] > 128 ? 256 : 128, 0, st>>>(
                    const_cast<float2*>(reinterpret_cast<const float2*>(in + ch.c_begin * cblk)),
                    at<float2>(w, o_mine[b]), static_cast<int>(lay.lp[i]), static_cast<int>(lay.mp[j]),
                    static_cast<int>(lay.l0(i)), static_cast<int>(lay.m0(j)), rowoff_me.p, tri_me);
                SPH_LAUNCH_CHECK();
                count_launch();
            }
            rec(eP1[b], st);
        };
        auto issue_a = [&](int64_t k) {
            const ShtChunk& ch = *chunks[k];
            const int b = k & 1;
            wait(cs, eP1[b]);
            if (k >= 2) wait(cs, eUC[b]);  // pay[b] consumed by chunk k-2's unpack
            alltoallv(comm->plane, q, ch.xia, at<float>(w, o_mine[b]), at<float>(w, o_pay[b]), cs);
            rec(eA1[b], cs);
            bytes_a += ch.bytes_ia;
        };
        pack_tri(0);
        issue_a(0);
        for (int64_t k = 0; k < n; ++k) {
            const ShtChunk& ch = *chunks[k];
            const int b = k & 1;
            const int64_t cq = ch.lay.cq(q);
            if (k + 1 < n) {
                // mine[(k+1)&1] was sent by chunk k-1's inbound exchange, which the caller's
                // stream waited for (eA1) before chunk k-1's unpack
                pack_tri(k + 1);
                issue_a(k + 1);
            }
            wait(st, eA1[b]);
            if (cq > 0) {
                {
                    ProfScope prof("dist_unpack_cint", st, 4.0 * ch.xia.recv_total() + 4.0 * sht->cint_elems(cq));
                    // two fields per CTA share the index math (as sht.cu's dense_to_cint)
                    dim3 g(static_cast<unsigned>((lay.mmax + 31) / 32), static_cast<unsigned>((lay.lmax + 63 + 63) / 64),
                           static_cast<unsigned>((cq + 1) / 2));
                    cint_unpack_kernel<2><<<g, 256, 0, st>>>(at<const float2>(w, o_pay[b]), cq,
                                                          static_cast<int>(lay.lmax), static_cast<int>(lay.mmax),
                                                          sht->Lp, pmap(ch.b0_ia), at<float>(w, o_cint));
                    SPH_LAUNCH_CHECK();
                    count_launch();
                }
                rec(eUC[b], st);
                if (ch.direct) {  // the unfold writes the outbound blocks in place
                    if (k >= 2) wait(st, eB2[b]);  // stage[b] sent by chunk k-2's outbound exchange
                    sht->inverse(at<float>(w, o_cint), cq, SPH_LAYOUT_INTERNAL, at<float>(w, o_stage[b]), w + o_shtws,
                                 st, ch.ring_b());
                } else {
                    sht->inverse(at<float>(w, o_cint), cq, SPH_LAYOUT_INTERNAL, at<float>(w, o_full), w + o_shtws, st);
                    if (k >= 2) wait(st, eB2[b]);  // stage[b] sent by chunk k-2's outbound exchange
                    ch.inv_pack.run(at<float>(w, o_full), at<float>(w, o_stage[b]), st, "dist_pack_fields");
                }
            } else {
                rec(eUC[b], st);
            }
            rec(eP2[b], st);
            wait(cs, eP2[b]);
            alltoallv(comm->plane, q, ch.xib, at<float>(w, o_stage[b]), y + ch.c_begin * fblk, cs);
            rec(eB2[b], cs);
            bytes_b += ch.bytes_ib;
        }
        rec(e_end, cs);
        wait(st, e_end);
        log("dist_isht", bytes_a);
        log("dist_isht", bytes_b);
    }
};

// ---------------------------------------------------------------- distributed DISCO
struct sph_dist_disco_plan_s {
    sph_comm comm = nullptr;
    sph::DiscoPlan* op = nullptr;
    sph::DiscoLayout lay;
    int64_t q = 0, i = 0, j = 0;
    sph::Exchange xh;
    sph::BoxList hpack, hunpack, rpack, runpack, mixbox;
    int64_t o_send = 0, o_recv = 0, o_rows = 0, o_mix = 0, o_part = 0, o_rss = 0, o_rsr = 0, o_dws = 0, total = 0;
    int64_t halo_bytes = 0, rs_bytes = 0;
    std::mutex mu;
    sph::DevBuf<uint8_t> own_ws;

    void create(sph_comm c, sph::DiscoPlan* p, int64_t cin, int64_t cout) {
        using namespace sph;
        require(cin >= 1 && cout >= 1, "dist_disco_apply: channel counts must be >= 1");
        comm = c;
        op = p;
        const int64_t nh = c->grid.sizes[2], nw = c->grid.sizes[3];
        lay = DiscoLayout(nh, nw, p->hin, p->win, p->hout, p->wout, cin, cout,
                          [p](int64_t a, int64_t n, int64_t* lo, int64_t* cnt) { p->input_rows(a, n, lo, cnt); });
        q = c->plane_rank;
        i = lay.pi(q);
        j = lay.pj(q);
        xh = lay.halo(q);
        DeviceGuard dg(p->device);
        hpack.set(lay.halo_pack(q));
        hunpack.set(lay.halo_unpack(q));
        const int64_t K = p->K, cz = lay.czp[j], mx = lay.rs_width();
        mixbox.set({{lay.cz0(j) * K, 0, 1, cout, cz * K, 0, cin * K, 0, cz * K}});
        if (nw > 1) {
            rpack.set(lay.rs_pack(q));
            runpack.set(lay.rs_unpack(q));
        }
        Carve cv;
        o_send = cv.take(4 * xh.send_total());
        o_recv = cv.take(4 * xh.recv_total());
        o_rows = cv.take(4 * cz * lay.needn[i] * lay.win);
        o_mix = cv.take(4 * cout * cz * K);
        o_part = cv.take(nw > 1 ? 4 * cout * lay.hop[i] * lay.wout : 0);
        o_rss = cv.take(nw > 1 ? 4 * nw * cout * lay.hop[i] * mx : 0);
        o_rsr = cv.take(nw > 1 ? 4 * cout * lay.hop[i] * mx : 0);
        o_dws = cv.take(cz ? p->rows_workspace_bytes(1, cz, cout, lay.needn[i], lay.hop[i]) : 0);
        total = cv.off;
        const int64_t planes = c->grid.sizes[0] * c->grid.sizes[1];
        halo_bytes = world_bytes(lay.P, planes, [&](int64_t r) { return lay.halo(r); });
        // reference accounting (distsim.hpp:262-266): every member receives its W_out slice
        // from the nw - 1 others
        rs_bytes = (nw - 1) * cout * lay.hout * lay.wout * 4 * planes;
    }
    uint8_t* ws_base(void* ws) {
        if (ws) return static_cast<uint8_t*>(ws);
        std::lock_guard<std::mutex> lk(mu);
        if (own_ws.n < static_cast<size_t>(total)) own_ws.alloc(total, true);
        return own_ws.p;
    }
    // x [C_in][H_i][W_j], mix [C_out][C_in][K] (replicated) -> y [C_out][Ho_i][Wo_j]
    void apply(const float* x, const float* mix, float* y, void* ws, cudaStream_t st) {
        using namespace sph;
        DeviceGuard dg(op->device);
        require_on_device(x, op->device, "dist_disco_apply");
        require_on_device(y, op->device, "dist_disco_apply");
        uint8_t* w = ws_base(ws);
        float* send = reinterpret_cast<float*>(w + o_send);
        float* recv = reinterpret_cast<float*>(w + o_recv);
        float* rows = reinterpret_cast<float*>(w + o_rows);
        float* mixs = reinterpret_cast<float*>(w + o_mix);
        const int64_t cz = lay.czp[j], nw = lay.nw;
        // A: channel slice x (filter-support rows) x full rings, one all-to-all of the plane
        hpack.run(x, send, st, "dist_pack_halo");
        alltoallv(comm->plane ? comm->plane : nullptr, q, xh, send, recv, st);
        {
            std::lock_guard<std::mutex> lk(comm->mu);
            comm->log.record("dist_disco", "polar+azimuth", "all_to_all", halo_bytes);
        }
        hunpack.run(recv, rows, st, "dist_unpack_halo");
        float* part = nw > 1 ? reinterpret_cast<float*>(w + o_part) : y;
        if (cz > 0) {
            mixbox.run(mix, mixs, st, "dist_mix_slice");
            op->apply_rows(rows, lay.need0[i], lay.needn[i], split_offset(lay.hop, i), lay.hop[i], mixs, 1, cz,
                           lay.cout, part, w + o_dws, st);
        } else {
            SPH_CUDA(cudaMemsetAsync(part, 0, 4 * lay.cout * lay.hop[i] * (nw > 1 ? lay.wout : lay.wop[j]), st));
        }
        if (nw > 1) {
            // sum the channel-slice partials over azimuth, scattered onto Wo_j
            float* rss = reinterpret_cast<float*>(w + o_rss);
            float* rsr = reinterpret_cast<float*>(w + o_rsr);
            rpack.run(part, rss, st, "dist_pack_rs");
            const int64_t cnt = lay.cout * lay.hop[i] * lay.rs_width();
            SPH_NCCL(sph::nccl().ReduceScatter(rss, rsr, static_cast<size_t>(cnt), ncclFloat, ncclSum, comm->az, st));
            runpack.run(rsr, y, st, "dist_unpack_rs");
        }
        std::lock_guard<std::mutex> lk(comm->mu);
        comm->log.record("dist_disco", "azimuth", "reduce_scatter", rs_bytes);
    }
};

// ------------------------------------------------------------------------ C ABI
namespace {
void write_out(const std::vector<int64_t>& v, int64_t* out, int64_t cap, int64_t* n) {
    sph::require(n != nullptr, "describe: null count pointer");
    *n = static_cast<int64_t>(v.size());
    if (out) {
        sph::require(cap >= *n, "describe: output buffer too small");
        std::memcpy(out, v.data(), sizeof(int64_t) * v.size());
    }
}
void put_exchange(std::vector<int64_t>& v, const sph::Exchange& x) {
    for (const auto* a : {&x.send_cnt, &x.send_off, &x.recv_cnt, &x.recv_off}) v.insert(v.end(), a->begin(), a->end());
}
void put_boxes(std::vector<int64_t>& v, const std::vector<sph::Box>& bs) {
    for (const auto& b : bs) v.insert(v.end(), {b.src_off, b.dst_off, b.n0, b.n1, b.n2, b.s0, b.s1, b.d0, b.d1});
}
}  // namespace

extern "C" {

int64_t sph_comm_id_bytes(void) { return static_cast<int64_t>(sizeof(ncclUniqueId)); }

int sph_comm_unique_id(void* id) {
    return guarded([&] {
        sph::require(id != nullptr, "comm: null id buffer");
        ncclUniqueId u;
        SPH_NCCL(sph::nccl().GetUniqueId(&u));
        std::memcpy(id, &u, sizeof(u));
    });
}

int sph_comm_create(const void* id, int64_t world, int64_t rank, const int64_t* sizes, sph_comm* comm) {
    return guarded([&] {
        sph::require(id && sizes && comm, "comm: null argument");
        auto h = std::make_unique<sph_comm_s>();
        for (int a = 0; a < 4; ++a) {
            sph::require(sizes[a] >= 1, "CommGrid: sizes must be >= 1");
            h->grid.sizes[a] = sizes[a];
        }
        sph::require(h->grid.world() == world, "comm: world size does not match the CommGrid");
        sph::require(rank >= 0 && rank < world, "comm: rank out of range");
        SPH_CUDA(cudaGetDevice(&h->device));
        h->rank = rank;
        h->coords = h->grid.coords(rank);
        const int64_t nh = sizes[2], nw = sizes[3];
        h->plane_size = nh * nw;
        h->plane_rank = h->coords[2] * nw + h->coords[3];
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        SPH_NCCL(sph::nccl().CommInitRank(&h->world, static_cast<int>(world), u, static_cast<int>(rank)));
        // plane: same (batch, ensemble); azimuth group: same (batch, ensemble, polar)
        const int plane_color = static_cast<int>(h->coords[0] * sizes[1] + h->coords[1]);
        // the plane's all-to-alls run beside compute kernels: bound their CTAs so the
        // distributed plans can leave exactly that many SMs free (GemmSmCap)
        if (const char* e = std::getenv("SPH_NCCL_MAX_CTAS")) h->nccl_ctas = std::max(1, std::atoi(e));
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.maxCTAs = h->nccl_ctas;
        SPH_NCCL(sph::nccl().CommSplit(h->world, plane_color, static_cast<int>(h->plane_rank), &h->plane, &cfg));
        SPH_NCCL(sph::nccl().CommSplit(h->world, static_cast<int>(plane_color * nh + h->coords[2]),
                               static_cast<int>(h->coords[3]), &h->az, nullptr));
        *comm = h.release();
    });
}

int sph_comm_destroy(sph_comm comm) {
    return guarded([&] { delete comm; });
}

int sph_comm_coords(sph_comm comm, int64_t* coords) {
    return guarded([&] {
        sph::require(comm && coords, "comm: null argument");
        for (int a = 0; a < 4; ++a) coords[a] = comm->coords[a];
    });
}

int sph_comm_traffic_csv(sph_comm comm, char* csv, size_t cap) {
    return guarded([&] {
        sph::require(comm && csv, "comm: null argument");
        std::lock_guard<std::mutex> lk(comm->mu);
        const std::string s = comm->log.csv();
        sph::require(s.size() + 1 <= cap, "traffic csv: buffer too small");
        std::memcpy(csv, s.c_str(), s.size() + 1);
    });
}

int sph_comm_traffic_reset(sph_comm comm) {
    return guarded([&] {
        sph::require(comm, "comm: null argument");
        std::lock_guard<std::mutex> lk(comm->mu);
        comm->log.recs.clear();
    });
}

int sph_dist_sht_plan_create(sph_comm comm, sph_sht_plan sht, int64_t C, sph_dist_sht_plan* plan) {
    return guarded([&] {
        sph::require(comm && sht && plan, "dist_sht: null argument");
        sph::require(sht->p.device == comm->device, "dist_sht: plan and communicator on different devices");
        auto h = std::make_unique<sph_dist_sht_plan_s>();
        h->create(comm, &sht->p, C);
        *plan = h.release();
    });
}

int sph_dist_sht_plan_destroy(sph_dist_sht_plan plan) {
    return guarded([&] { delete plan; });
}

int sph_dist_sht_local(sph_dist_sht_plan plan, int64_t* info) {
    return guarded([&] {
        sph::require(plan && info, "dist_sht: null argument");
        const auto& L = plan->lay;
        const int64_t v[10] = {L.h0(plan->i), L.hp[plan->i], L.w0(plan->j), L.wp[plan->j], L.l0(plan->i),
                               L.lp[plan->i], L.m0(plan->j),  L.mp[plan->j], L.c0(plan->q), L.cq(plan->q)};
        std::memcpy(info, v, sizeof(v));
    });
}

int64_t sph_dist_sht_workspace_bytes(sph_dist_sht_plan plan) { return plan ? plan->total : -1; }

int sph_dist_sht_forward(sph_dist_sht_plan plan, const float* x, float* coeffs, void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "dist_sht_forward: null plan");
        plan->forward(x, coeffs, workspace, S(stream));
    });
}

int sph_dist_sht_inverse(sph_dist_sht_plan plan, const float* coeffs, float* y, void* workspace, void* stream) {
    return guarded([&] {
        sph::require(plan, "dist_sht_inverse: null plan");
        plan->inverse(coeffs, y, workspace, S(stream));
    });
}

int sph_dist_disco_plan_create(sph_comm comm, sph_disco_plan op, int64_t c_in, int64_t c_out,
                               sph_dist_disco_plan* plan) {
    return guarded([&] {
        sph::require(comm && op && plan, "dist_disco: null argument");
        sph::require(op->p.device == comm->device, "dist_disco: plan and communicator on different devices");
        auto h = std::make_unique<sph_dist_disco_plan_s>();
        h->create(comm, &op->p, c_in, c_out);
        *plan = h.release();
    });
}

int sph_dist_disco_plan_destroy(sph_dist_disco_plan plan) {
    return guarded([&] { delete plan; });
}

int sph_dist_disco_local(sph_dist_disco_plan plan, int64_t* info) {
    return guarded([&] {
        sph::require(plan && info, "dist_disco: null argument");
        const auto& L = plan->lay;
        const int64_t i = plan->i, j = plan->j;
        const int64_t v[12] = {L.h0(i), L.hp[i], L.w0(j), L.wp[j], sph::split_offset(L.hop, i), L.hop[i],
                               sph::split_offset(L.wop, j), L.wop[j], L.cz0(j), L.czp[j], L.need0[i], L.needn[i]};
        std::memcpy(info, v, sizeof(v));
    });
}

int64_t sph_dist_disco_workspace_bytes(sph_dist_disco_plan plan) { return plan ? plan->total : -1; }

int sph_dist_disco_apply(sph_dist_disco_plan plan, const float* x, const float* mix, float* y, void* workspace,
                         void* stream) {
    return guarded([&] {
        sph::require(plan, "dist_disco_apply: null plan");
        plan->apply(x, mix, y, workspace, S(stream));
    });
}

// Host-only schedule descriptions (no GPU, no NCCL): what = 0 ranges
// (h0,hn,w0,wn,l0,ln,m0,mn,c0,cn); 1..4 exchanges fwd_fields, fwd_coeffs, inv_coeffs,
// inv_fields as [send_cnt|send_off|recv_cnt|recv_off] x P; 5 / 6 the fwd_unpack / inv_pack
// boxes (9 int64 each); 7 rowoff of the rank's own coefficient block.
int sph_dist_sht_describe(int64_t nh, int64_t nw, int64_t q, int64_t nlat, int64_t nlon, int64_t lmax,
                          int64_t mmax, int64_t C, int what, int64_t* out, int64_t cap, int64_t* n) {
    return guarded([&] {
        const sph::ShtLayout L(nh, nw, nlat, nlon, lmax, mmax, C);
        sph::require(q >= 0 && q < L.P, "describe: rank out of range");
        std::vector<int64_t> v;
        const int64_t i = L.pi(q), j = L.pj(q);
        switch (what) {
            case 0: v = {L.h0(i), L.hp[i], L.w0(j), L.wp[j], L.l0(i), L.lp[i], L.m0(j), L.mp[j], L.c0(q), L.cq(q)}; break;
            case 1: put_exchange(v, L.fwd_fields(q)); break;
            case 2: put_exchange(v, L.fwd_coeffs(q)); break;
            case 3: put_exchange(v, L.inv_coeffs(q)); break;
            case 4: put_exchange(v, L.inv_fields(q)); break;
            case 5: put_boxes(v, L.fwd_unpack(q)); break;
            case 6: put_boxes(v, L.inv_pack(q)); break;
            case 7: v = L.rowoff(q); break;
            default: sph::require(false, "describe: unknown item");
        }
        write_out(v, out, cap, n);
    });
}

// what = 0 ranges (h0,hn,w0,wn,ho0,hon,wo0,won,cz0,czn,need0,needn); 1 halo exchange;
// 2 / 3 halo pack / unpack boxes; 4 / 5 reduce-scatter pack / unpack boxes; 6 rs slot width.
// band_lo / band_n: input row band of every output row (the plan's filter support).
int sph_dist_disco_describe(int64_t nh, int64_t nw, int64_t q, int64_t hin, int64_t win, int64_t hout, int64_t wout,
                            int64_t cin, int64_t cout, const int64_t* band_lo, const int64_t* band_n, int what,
                            int64_t* out, int64_t cap, int64_t* n) {
    return guarded([&] {
        sph::require(band_lo && band_n, "describe: null band arrays");
        const sph::DiscoLayout L(nh, nw, hin, win, hout, wout, cin, cout,
                                 [&](int64_t a, int64_t cnt, int64_t* lo, int64_t* nn) {
                                     int64_t l = band_lo[a], h = band_lo[a] + band_n[a];
                                     for (int64_t r = a; r < a + cnt; ++r) {
                                         l = std::min(l, band_lo[r]);
                                         h = std::max(h, band_lo[r] + band_n[r]);
                                     }
                                     *lo = l;
                                     *nn = h - l;
                                 });
        sph::require(q >= 0 && q < L.P, "describe: rank out of range");
        std::vector<int64_t> v;
        const int64_t i = L.pi(q), j = L.pj(q);
        switch (what) {
            case 0:
                v = {L.h0(i),   L.hp[i],   L.w0(j),  L.wp[j],  sph::split_offset(L.hop, i), L.hop[i],
                     sph::split_offset(L.wop, j), L.wop[j], L.cz0(j), L.czp[j], L.need0[i], L.needn[i]};
                break;
            case 1: put_exchange(v, L.halo(q)); break;
            case 2: put_boxes(v, L.halo_pack(q)); break;
            case 3: put_boxes(v, L.halo_unpack(q)); break;
            case 4: put_boxes(v, L.rs_pack(q)); break;
            case 5: put_boxes(v, L.rs_unpack(q)); break;
            case 6: v = {L.rs_width()}; break;
            default: sph::require(false, "describe: unknown item");
        }
        write_out(v, out, cap, n);
    });
}

}  // extern "C"
