// Spectral convolution (convolution.hpp:286-304) and the neural-operator block
// epilogue (model.hpp:355-368), both on the shared tcgen05 grouped-GEMM engine.
#include <algorithm>

#include <mutex>

#include "disco.cuh"

namespace sph {

namespace {

__device__ __forceinline__ float gelu_erfc(float x) {  // model.hpp:42-44
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

// kernel [cout][cin][klmax] -> Kt hi/lo [(l*cout + o)][ldk], l < lmax (tiled transpose)
__global__ void kernel_transpose_split(const float* __restrict__ k, int64_t cout, int64_t cin,
                                       int64_t klmax, int64_t lmax, int64_t ldk,
                                       float* __restrict__ hi, float* __restrict__ lo) {
    __shared__ float tile[32][33];
    const int64_t o = blockIdx.z;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32, l0 = static_cast<int64_t>(blockIdx.y) * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, l = l0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < cin && l < lmax) ? k[(o * cin + i) * klmax + l] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t l = l0 + r, i = i0 + threadIdx.x;
        if (l < lmax && i < ldk) {
            const float x = i < cin ? tile[threadIdx.x][r] : 0.f;
            uint32_t u;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
            const float h = __uint_as_float(u);
            const int64_t idx = (l * cout + o) * ldk + i;
            hi[idx] = h;
            lo[idx] = x - h;
        }
    }
}

// C_int (F = B*cin fields) -> Xg[row_off[l] + (m*2 + reim)*B + b][i]
// C_int [(m*2+p)][2F (b, i, re/im)][Lp] <-> per-l GEMM rows: 32 x 32 tiled transposes over
// (channel, lp) for one (m, p, b, re/im) -- both sides in 128-byte runs (the element-wise
// forms read with a stride of 2*Lp resp. ldy floats).  blockIdx.z = ((m*2 + p)*B + b)*2 + re/im.
// Xg[row_off[l] + (m*2+reim)*B + b][i] = C_int(l, m; b, i, reim)  (l = m + p + 2 lp)
__global__ void spec_gather_kernel(const float* __restrict__ cint, const int64_t* __restrict__ row_off,
                                   int64_t lmax, int64_t B, int64_t cin, int Lp, int64_t ldx,
                                   float* __restrict__ Xg) {
    __shared__ float t[32][33];
    int64_t z = blockIdx.z;
    const int reim = static_cast<int>(z & 1);
    z >>= 1;
    const int64_t b = z % B;
    z /= B;
    const int p = static_cast<int>(z & 1);
    const int64_t m = z >> 1;
    const int64_t twoF = 2 * B * cin;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32, lp0 = static_cast<int64_t>(blockIdx.y) * 32;
    const int64_t nlp = (lmax - m - p + 1) / 2;  // lp with l = m + p + 2 lp < lmax
    if (lp0 >= nlp) return;                      // no GEMM rows in this tile (the triangle)
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int64_t i = i0 + r, lp = lp0 + threadIdx.x;
        t[r][threadIdx.x] =
            (i < cin && lp < nlp) ? __ldg(cint + ((m * 2 + p) * twoF + 2 * (b * cin + i) + reim) * Lp + lp) : 0.f;
    }
    __syncthreads();
    // the 4 row offsets of this thread first (one dependent-load round instead of four)
    int64_t ro[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t lp = lp0 + threadIdx.y + 8 * k, l = m + p + 2 * lp;
        ro[k] = (lp < Lp && l < lmax) ? __ldg(row_off + l) : -1;
    }
    const int64_t i = i0 + threadIdx.x;
    if (i >= ldx) return;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (ro[k] < 0) continue;
        const int64_t row = ro[k] + (m * 2 + reim) * B + b;
        Xg[row * ldx + i] = i < cin ? t[threadIdx.x][threadIdx.y + 8 * k] : 0.f;
    }
}

// Yg[row_off[l] + (m*2+reim)*B + b][o] -> C_int (F = B*cout) incl. zero padding
__global__ void spec_scatter_kernel(const float* __restrict__ Yg, const int64_t* __restrict__ row_off,
                                    int64_t lmax, int64_t B, int64_t cout, int Lp, int64_t ldy,
                                    float* __restrict__ cint) {
    __shared__ float t[32][33];
    int64_t z = blockIdx.z;
    const int reim = static_cast<int>(z & 1);
    z >>= 1;
    const int64_t b = z % B;
    z /= B;
    const int p = static_cast<int>(z & 1);
    const int64_t m = z >> 1;
    const int64_t twoF = 2 * B * cout;
    const int64_t o0 = static_cast<int64_t>(blockIdx.x) * 32, lp0 = static_cast<int64_t>(blockIdx.y) * 32;
    {  // row offsets, then the 4 row loads, before any shared-memory store
        const int64_t o = o0 + threadIdx.x;
        int64_t ro[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t lp = lp0 + threadIdx.y + 8 * k, l = m + p + 2 * lp;
            ro[k] = (lp < Lp && l < lmax && o < cout) ? __ldg(row_off + l) : -1;
        }
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            v[k] = ro[k] >= 0 ? __ldg(Yg + (ro[k] + (m * 2 + reim) * B + b) * ldy + o) : 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) t[threadIdx.y + 8 * k][threadIdx.x] = v[k];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int64_t o = o0 + r, lp = lp0 + threadIdx.x;
        if (o < cout && lp < Lp) cint[((m * 2 + p) * twoF + 2 * (b * cout + o) + reim) * Lp + lp] = t[threadIdx.x][r];
    }
}

// G[(b*P + p)][c] = gelu(conv[b][c][p])  (tiled transpose)
// 32 x 32 tiles, GELU_PT consecutive point tiles per CTA (amortises the CTA set-up of a
// 4-element-per-thread tile over 4x the bytes)
constexpr int GELU_PT = 4;
__global__ void gelu_transpose_kernel(const float* __restrict__ conv, int64_t C, int64_t P,
                                      int64_t ldc, float* __restrict__ G) {
    __shared__ float tile[32][33];
    const int64_t b = blockIdx.z;
    const int64_t c0 = static_cast<int64_t>(blockIdx.y) * 32;
    const float* cb = conv + (b * C + c0) * P;
    float* gb = G + b * P * ldc + c0;
    for (int pt = 0; pt < GELU_PT; ++pt) {
        const int64_t p0 = (static_cast<int64_t>(blockIdx.x) * GELU_PT + pt) * 32;
        if (p0 >= P) break;
        if (pt) __syncthreads();
#pragma unroll
        for (int r = threadIdx.y; r < 32; r += 8) {
            const int64_t p = p0 + threadIdx.x;
            tile[r][threadIdx.x] = (c0 + r < C && p < P) ? gelu_erfc(__ldg(cb + r * P + p)) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int r = threadIdx.y; r < 32; r += 8) {
            const int64_t p = p0 + r;
            const int64_t c = c0 + threadIdx.x;
            if (p < P && c < ldc) gb[p * ldc + threadIdx.x] = c < C ? tile[threadIdx.x][r] : 0.f;
        }
    }
}

// y = x + scale[c] (y + b2[c]); grid (point chunks, c, b), float4 when P % 4 == 0
// P % 4 == 0: one 32-channel x 128-point tile per CTA, float4 point loads (all four per
// thread in flight), a single barrier, float4 channel stores of the transposed rows; tile
// pitch 129 keeps the column reads conflict-free
__global__ void __launch_bounds__(256) gelu_transpose4_kernel(const float* __restrict__ conv, int64_t C, int64_t P,
                                                              int64_t ldc, float* __restrict__ G) {
    __shared__ float tile[32][129];
    const int64_t b = blockIdx.z;
    const int64_t c0 = static_cast<int64_t>(blockIdx.y) * 32, p0 = static_cast<int64_t>(blockIdx.x) * 128;
    const int t = threadIdx.x;
    float4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int idx = t + 256 * i;
        const int c = idx >> 5, p4 = 4 * (idx & 31);
        v[i] = (c0 + c < C && p0 + p4 < P)
                   ? __ldg(reinterpret_cast<const float4*>(conv + (b * C + c0 + c) * P + p0 + p4))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int idx = t + 256 * i;
        const int c = idx >> 5, p4 = 4 * (idx & 31);
        const bool ok = c0 + c < C;
        tile[c][p4] = ok ? gelu_erfc(v[i].x) : 0.f;
        tile[c][p4 + 1] = ok ? gelu_erfc(v[i].y) : 0.f;
        tile[c][p4 + 2] = ok ? gelu_erfc(v[i].z) : 0.f;
        tile[c][p4 + 3] = ok ? gelu_erfc(v[i].w) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int idx = t + 256 * i;
        const int pr = idx >> 3, q = idx & 7;
        const int64_t p = p0 + pr;
        if (p >= P || c0 + 4 * q >= ldc) continue;
        const float4 o = make_float4(tile[4 * q][pr], tile[4 * q + 1][pr], tile[4 * q + 2][pr], tile[4 * q + 3][pr]);
        *reinterpret_cast<float4*>(G + (b * P + p) * ldc + c0 + 4 * q) = o;
    }
}

__global__ void residual_kernel(float* __restrict__ y, const float* __restrict__ x, int64_t B,
                                int64_t C, int64_t P, const float* __restrict__ b2,
                                const float* __restrict__ scales) {
    const int64_t c = blockIdx.y, b = blockIdx.z;
    const float s = scales[c], bb = b2[c];
    const int64_t base = (b * C + c) * P;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if ((P & 3) == 0) {
        float4* y4 = reinterpret_cast<float4*>(y + base);
        const float4* x4 = reinterpret_cast<const float4*>(x + base);
        for (int64_t i = t0; i < P / 4; i += stride) {
            const float4 xv = __ldg(x4 + i);
            float4 yv = y4[i];
            yv.x = xv.x + s * (yv.x + bb);
            yv.y = xv.y + s * (yv.y + bb);
            yv.z = xv.z + s * (yv.z + bb);
            yv.w = xv.w + s * (yv.w + bb);
            y4[i] = yv;
        }
    } else {
        for (int64_t i = t0; i < P; i += stride) y[base + i] = x[base + i] + s * (y[base + i] + bb);
    }
}


struct SpecProblem {
    std::vector<int64_t> row_off;
    std::vector<int32_t> row_l;
    DevBuf<int64_t> d_row_off;
    DevBuf<int32_t> d_row_l;
    int64_t nrows = 0;
    GroupedGemm gemm;
};

std::mutex g_mu;
// keyed by the plan's address AND its truncation: a plan created later at a freed plan's
// address must not inherit its per-degree tile list
std::map<std::tuple<const void*, int64_t, int64_t, int64_t, int64_t, int64_t>, std::unique_ptr<SpecProblem>> g_spec;
std::map<std::tuple<int64_t, int64_t, int64_t, int64_t, int>, std::unique_ptr<GroupedGemm>> g_mlp;

struct SpecWs {
    int64_t ldx, ldy, cin_off, cout_off, x_off, y_off, khi_off, klo_off, sht_off, total;
};
SpecWs spec_ws(const ShtPlan& p, int64_t B, int64_t cin, int64_t cout) {
    SpecWs w;
    w.ldx = static_cast<int64_t>(round_up(cin, 4));
    w.ldy = static_cast<int64_t>(round_up(cout, 4));
    int64_t nrows = 0;
    for (int64_t l = 0; l < p.lmax; ++l) nrows += 2 * B * (std::min(l, p.mmax - 1) + 1);
    int64_t o = 0;
    w.cin_off = o;  o += round_up(p.cint_elems(B * cin) * 4, 256);
    w.cout_off = o; o += round_up(p.cint_elems(B * cout) * 4, 256);
    w.x_off = o;    o += round_up(nrows * w.ldx * 4, 256);
    w.y_off = o;    o += round_up(nrows * w.ldy * 4, 256);
    w.khi_off = o;  o += round_up(p.lmax * cout * w.ldx * 4, 256);
    w.klo_off = o;  o += round_up(p.lmax * cout * w.ldx * 4, 256);
    w.sht_off = o;  o += round_up(std::max(p.workspace_bytes(B * cin), p.workspace_bytes(B * cout)), 256);
    w.total = o;
    return w;
}

}  // namespace

int64_t spectral_conv_ws_bytes(const ShtPlan& p, int64_t B, int64_t cin, int64_t cout) {
    return spec_ws(p, B, cin, cout).total;
}

namespace {
// y(o,l,m) = sum_i c(i,l,m) k(o,i,l)  (convolution.hpp:295-302) on the GEMM-native C_int
// layout of the plan: gather per degree l into [(m, re/im, b)][c_in] rows, one grouped
// tcgen05 GEMM over l with the kernel transposed to [l][c_out][c_in], scatter back.
void spectral_mix_cint(ShtPlan& p, const float* cin_i, const float* kernel, int64_t B, int64_t cin,
                       int64_t cout, int64_t klmax, float* cout_i, uint8_t* base, const SpecWs& w,
                       cudaStream_t st) {
    const int64_t lmax = p.lmax, mmax = p.mmax;
    float* Xg = reinterpret_cast<float*>(base + w.x_off);
    float* Yg = reinterpret_cast<float*>(base + w.y_off);
    float* khi = reinterpret_cast<float*>(base + w.khi_off);
    float* klo = reinterpret_cast<float*>(base + w.klo_off);
    SpecProblem* sp;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto& slot = g_spec[std::make_tuple(static_cast<const void*>(&p), B, cin, cout, p.lmax, p.mmax)];
        if (!slot) {
            auto s = std::make_unique<SpecProblem>();
            s->row_off.assign(lmax + 1, 0);
            for (int64_t l = 0; l < lmax; ++l)
                s->row_off[l + 1] = s->row_off[l] + 2 * B * (std::min(l, mmax - 1) + 1);
            s->nrows = s->row_off[lmax];
            s->row_l.resize(s->nrows);
            for (int64_t l = 0; l < lmax; ++l)
                for (int64_t r = s->row_off[l]; r < s->row_off[l + 1]; ++r) s->row_l[r] = static_cast<int32_t>(l);
            s->d_row_off.alloc(s->row_off.size(), false);
            SPH_CUDA(cudaMemcpy(s->d_row_off.p, s->row_off.data(), s->row_off.size() * 8, cudaMemcpyHostToDevice));
            s->d_row_l.alloc(std::max<size_t>(s->row_l.size(), 1), false);
            SPH_CUDA(cudaMemcpy(s->d_row_l.p, s->row_l.data(), s->row_l.size() * 4, cudaMemcpyHostToDevice));
            GroupedGemm& g = s->gemm;
            g.A = {nullptr, s->nrows, cin, w.ldx};
            g.Bhi = {nullptr, lmax * cout, cin, w.ldx};
            g.Blo = {nullptr, lmax * cout, cin, w.ldx};
            g.store = STORE_ROW;
            g.bn = cout >= 256 ? 256 : 128;
            g.name = "gemm_spectral_mix";
            g.cluster = 1;  // per-degree groups: 0.152 ms vs 0.174 ms at 2 (cfg4)
            for (int64_t l = 0; l < lmax; ++l) {
                GemmGroup gr;
                gr.a_row0 = static_cast<int32_t>(s->row_off[l]);
                gr.b_row0 = static_cast<int32_t>(l * cout);
                gr.M = static_cast<int32_t>(s->row_off[l + 1] - s->row_off[l]);
                gr.N = static_cast<int32_t>(cout);
                gr.K = static_cast<int32_t>(cin);
                gr.ldd = static_cast<int32_t>(w.ldy);
                gr.zero_to = 0;
                gr.d_off = s->row_off[l] * w.ldy;
                g.groups.push_back(gr);
            }
            g.finalize();
            slot = std::move(s);
        }
        sp = slot.get();
    }
    dim3 grid(static_cast<unsigned>((w.ldx + 31) / 32), static_cast<unsigned>((lmax + 31) / 32),
              static_cast<unsigned>(cout));
    {
        ProfScope prof("spectral_kernel_split", st);
        kernel_transpose_split<<<grid, dim3(32, 8), 0, st>>>(kernel, cout, cin, klmax, lmax, w.ldx, khi, klo);
        SPH_LAUNCH_CHECK();
    }
    {
        ProfScope prof("spectral_gather", st);
        require(mmax * 4 * B <= 65535, "spectral_conv: too many orders x batches for the gather grid");
        dim3 tg(static_cast<unsigned>((w.ldx + 31) / 32), static_cast<unsigned>((p.Lp + 31) / 32),
                static_cast<unsigned>(mmax * 4 * B));
        spec_gather_kernel<<<tg, dim3(32, 8), 0, st>>>(cin_i, sp->d_row_off.p, lmax, B, cin, p.Lp, w.ldx, Xg);
        SPH_LAUNCH_CHECK();
    }
    count_launch(2);
    gemm_run(sp->gemm, Xg, Yg, p.prec, st, khi, klo);
    {
        ProfScope prof("spectral_scatter", st);
        dim3 ts(static_cast<unsigned>((cout + 31) / 32), static_cast<unsigned>((p.Lp + 31) / 32),
                static_cast<unsigned>(mmax * 4 * B));
        spec_scatter_kernel<<<ts, dim3(32, 8), 0, st>>>(Yg, sp->d_row_off.p, lmax, B, cout, p.Lp, w.ldy, cout_i);
        SPH_LAUNCH_CHECK();
    }
    count_launch();
}
}  // namespace

void spectral_conv(ShtPlan& p, const float* x, const float* kernel, int64_t B, int64_t cin,
                   int64_t cout, int64_t klmax, float* y, void* ws, cudaStream_t st) {
    require(p.kind == SPH_GAUSSIAN, "spectral_conv: requires a gaussian grid");  // :287-288
    require(cin >= 1 && cout >= 1 && klmax >= 1, "spectral_conv: kernel channel mismatch");
    const int64_t lmax = std::min<int64_t>(klmax, p.nlat);
    const int64_t mmax = std::min<int64_t>(lmax, p.nlon / 2);
    require(p.lmax == lmax && p.mmax == mmax,
            "spectral_conv: plan truncation must be lmax=min(klmax,nlat), mmax=min(lmax,nlon/2)");
    if (B == 0) return;
    DeviceGuard dguard(p.device);
    const SpecWs w = spec_ws(p, B, cin, cout);
    uint8_t* base = static_cast<uint8_t*>(ws);
    DevBuf<uint8_t> tmp;
    if (!base) {
        tmp.alloc(w.total, false);
        base = tmp.p;
    }
    float* cin_i = reinterpret_cast<float*>(base + w.cin_off);
    float* cout_i = reinterpret_cast<float*>(base + w.cout_off);
    void* sws = base + w.sht_off;
    // 1. forward SHT of the B*cin input fields (convolution.hpp:294)
    p.forward(x, B * cin, cin_i, SPH_LAYOUT_INTERNAL, sws, st);
    // 2. the per-degree channel mix (convolution.hpp:295-302)
    spectral_mix_cint(p, cin_i, kernel, B, cin, cout, klmax, cout_i, base, w, st);
    // 3. inverse SHT (convolution.hpp:303)
    p.inverse(cout_i, B * cout, SPH_LAYOUT_INTERNAL, y, sws, st);
    if (tmp.p) SPH_CUDA(cudaStreamSynchronize(st));
}

void spectral_mix(ShtPlan& p, const float* coeffs, const float* kernel, int64_t B, int64_t cin, int64_t cout,
                  int64_t klmax, float* out, void* ws, cudaStream_t st) {
    require(cin >= 1 && cout >= 1, "spectral_mix: kernel channel mismatch");
    require(klmax >= p.lmax, "spectral_mix: kernel must cover every degree of the coefficients");
    if (B == 0) return;
    DeviceGuard dguard(p.device);
    require_on_device(coeffs, p.device, "spectral_mix");
    require_on_device(out, p.device, "spectral_mix");
    const SpecWs w = spec_ws(p, B, cin, cout);
    uint8_t* base = static_cast<uint8_t*>(ws);
    DevBuf<uint8_t> tmp;
    if (!base) {
        tmp.alloc(w.total, false);
        base = tmp.p;
    }
    float* cin_i = reinterpret_cast<float*>(base + w.cin_off);
    float* cout_i = reinterpret_cast<float*>(base + w.cout_off);
    dense_to_cint(p, coeffs, B * cin, cin_i, st);
    spectral_mix_cint(p, cin_i, kernel, B, cin, cout, klmax, cout_i, base, w, st);
    cint_to_dense(p, cout_i, B * cout, 0, p.mmax, p.mmax, out, st);
    if (tmp.p) SPH_CUDA(cudaStreamSynchronize(st));
}

void block_epilogue(const float* conv, const float* x, const float* w1, const float* b1,
                    const float* w2, const float* b2, const float* scales, int64_t B, int64_t C,
                    int64_t H, int64_t P, float* y, cudaStream_t st) {
    require(B >= 0 && C >= 1 && H >= 1 && P >= 0, "block_apply: bad shapes");
    if (B == 0 || P == 0) return;
    const int prec = SPH_PREC_3XTF32;
    const int64_t ldc = static_cast<int64_t>(round_up(C, 4)), ldh = static_cast<int64_t>(round_up(H, 4));
    // workspace: G [B*P][ldc], Hm [B*P][ldh], W1 hi/lo [H][ldc], W2 hi/lo [C][ldh]
    const int64_t nG = B * P * ldc, nH = B * P * ldh, nW1 = H * ldc, nW2 = C * ldh;
    require(B <= 65535 && C <= 65535, "block_apply: too many channels / batches");
    require(B * P < (1LL << 31), "block: too many points");
    // stream-ordered workspace from the library's own pool (release threshold UINT64_MAX
    // keeps the ~0.8 GB resident across synchronisations; the device's default pool,
    // which other cudaMallocAsync users share, is left untouched).  The guard returns
    // it to the pool on every exit path, errors included.
    StreamBuf wsb(4 * (nG + nH + 2 * nW1 + 2 * nW2) + 1024, st);
    float* wsp = static_cast<float*>(wsb.p);
    float* G = wsp;
    float* Hm = G + round_up(nG, 64);
    float* w1h = Hm + round_up(nH, 64);
    float* w1l = w1h + round_up(nW1, 64);
    float* w2h = w1l + round_up(nW1, 64);
    float* w2l = w2h + round_up(nW2, 64);
    GroupedGemm *g1, *g2;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto& s1 = g_mlp[std::make_tuple(B, C, H, P, 1)];
        if (!s1) {
            auto g = std::make_unique<GroupedGemm>();
            g->A = {nullptr, B * P, C, ldc};
            g->Bhi = {nullptr, H, C, ldc};
            g->Blo = {nullptr, H, C, ldc};
            g->store = STORE_ROW;
            g->bn = H >= 256 ? 256 : 128;
            g->name = "gemm_mlp1";
            static const int row_tma = std::getenv("SPH_MLP_ROW_TMA") ? std::atoi(std::getenv("SPH_MLP_ROW_TMA")) : 1;
            g->row_tma = row_tma != 0;
            g->groups.push_back({0, 0, static_cast<int32_t>(B * P), static_cast<int32_t>(H),
                                 static_cast<int32_t>(C), static_cast<int32_t>(ldh), 0, 0});
            g->finalize();
            s1 = std::move(g);
        }
        auto& s2 = g_mlp[std::make_tuple(B, C, H, P, 2)];
        if (!s2) {
            auto g = std::make_unique<GroupedGemm>();
            g->A = {nullptr, B * P, H, ldh};
            g->Bhi = {nullptr, C, H, ldh};
            g->Blo = {nullptr, C, H, ldh};
            g->store = STORE_TRANS;
            g->bn = C >= 256 ? 256 : 128;
            g->name = "gemm_mlp2";
            for (int64_t b = 0; b < B; ++b)
                g->groups.push_back({static_cast<int32_t>(b * P), 0, static_cast<int32_t>(P),
                                     static_cast<int32_t>(C), static_cast<int32_t>(H),
                                     static_cast<int32_t>(P), 0, b * C * P});
            g->finalize();
            s2 = std::move(g);
        }
        g1 = s1.get();
        g2 = s2.get();
    }
    split_rows(w1, H, C, ldc, w1h, w1l, st);
    split_rows(w2, C, H, ldh, w2h, w2l, st);
    dim3 grid(static_cast<unsigned>((P + 32 * GELU_PT - 1) / (32 * GELU_PT)), static_cast<unsigned>((ldc + 31) / 32),
              static_cast<unsigned>(B));
    {
        ProfScope prof("mlp_gelu_transpose", st);
        if (P % 4 == 0 && ldc % 32 == 0 && (reinterpret_cast<uintptr_t>(conv) & 15) == 0) {
            dim3 g4(static_cast<unsigned>((P + 127) / 128), static_cast<unsigned>(ldc / 32), static_cast<unsigned>(B));
            gelu_transpose4_kernel<<<g4, 256, 0, st>>>(conv, C, P, ldc, G);
        } else {
            gelu_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(conv, C, P, ldc, G);
        }
        SPH_LAUNCH_CHECK();
    }
    count_launch();
    // bias + GeLU fused into the first layer's epilogue (cfg4 block pair: 1.03 + 1.04 ms as
    // GEMM + elementwise pass -> 1.73 ms fused).  The layer-scaled residual stays a separate
    // pass: fused into the second layer's epilogue (GemmEpi mode 2) it measured 1.50 ms vs
    // 0.67 + 0.53 -- each output chunk waits on HBM reads of the residual.
    GemmEpi e1;
    e1.mode = 1;
    e1.bias = b1;
    gemm_run(*g1, G, Hm, prec, st, w1h, w1l, &e1);
    gemm_run(*g2, Hm, y, prec, st, w2h, w2l);
    {
        ProfScope prof("mlp_residual", st);
        const int64_t chunks = std::min<int64_t>((P / 4 + 255) / 256 + 1, 64);
        residual_kernel<<<dim3(static_cast<unsigned>(chunks), static_cast<unsigned>(C), static_cast<unsigned>(B)), 256, 0,
                          st>>>(y, x, B, C, P, b2, scales);
        SPH_LAUNCH_CHECK();
    }
    count_launch();
}

}  // namespace sph
