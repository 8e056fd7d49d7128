/* sphere_gpu.h -- C ABI of the B200-native spherical-operator hot path (libsphgpu.so).
 *
 * Drop-in for the operator API of the reference library spheretk
 * (/root/reference/proj/include/sphere/, namespace sphere).  Each entry point names the
 * reference function it replaces (file:line).  Conventions:
 *   - every call returns an int status (SPH_OK or an error code); the message of the
 *     last failure on the calling thread is available from sph_last_error();
 *   - plans are immutable after creation and may be shared between threads; execute
 *     calls are stream-ordered (cudaStream_t passed as void*, NULL = legacy stream);
 *   - the caller owns every data buffer.  Unless stated otherwise data pointers are
 *     DEVICE pointers of the current device, fp32, in the reference layouts:
 *         fields  [F][nlat][nlon]                 (field.hpp:15-35, F = batch*channels)
 *         coeffs  [F][lmax][mmax] complex64       (harmonics.hpp:24-42, zeros above
 *                                                  the diagonal) for SPH_LAYOUT_DENSE_LM
 *         mix     [c_out][c_in][K]                (convolution.hpp:126-139)
 *   - `lmax` / `mmax` are COUNTS as in the reference (degrees 0..lmax-1,
 *     harmonics.hpp:25-26).
 * No torch types, no C++ types: plain pointers and sizes.
 */
#ifndef SPHERE_GPU_H
#define SPHERE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror the reference's exception classes) ---------------- */
#define SPH_OK 0
#define SPH_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define SPH_ERR_RUNTIME 2          /* std::runtime_error (e.g. grid.hpp:117-119) */
#define SPH_ERR_CUDA 3
#define SPH_ERR_NCCL 4
#define SPH_ERR_OOM 5

/* ---- enums ------------------------------------------------------------------- */
#define SPH_EQUIANGULAR 0 /* grid.hpp:69  build_equiangular */
#define SPH_GAUSSIAN 1    /* grid.hpp:91  build_gaussian    */

/* precision of the tensor-core contractions (Legendre, channel mixes) */
#define SPH_PREC_3XTF32 0   /* default: hi*hi + hi*lo + lo*hi on tcgen05, fp32 accum */
#define SPH_PREC_TF32 1     /* reduced-precision mode: one tcgen05 tf32 MMA (~1e-3)  */
#define SPH_PREC_FP32_SIMT 2 /* fp32 FMA SIMT kernels (parity anchor)                */

/* plan flags */
#define SPH_FLAG_PREC_MASK 0x3
/* sharp edge of the reference: sht_forward throws on equiangular grids
 * (harmonics.hpp:129-130); the reference's equiangular forward is dist_sht_forward
 * (distsim.hpp:404).  Plans created without this flag reject equiangular forwards. */
#define SPH_FLAG_ALLOW_EQUIANGULAR_FORWARD 0x10
/* adjoint plan (the SHT's backward pass; no reference counterpart):
 * under the real inner product <c, d> = sum Re(conj(c) d) over the stored m >= 0,
 * sph_sht_forward computes the adjoint of sht_inverse (grid field -> coefficients:
 * unweighted analysis, m >= 1 doubled; any grid kind) and sph_sht_inverse computes the
 * adjoint of sht_forward (coefficients -> field: quadrature-weighted synthesis with
 * m >= 1 halved).  Same kernels, different tables. */
#define SPH_FLAG_ADJOINT 0x20

/* coefficient layouts */
#define SPH_LAYOUT_DENSE_LM 0 /* reference [F][lmax][mmax] complex64 */
#define SPH_LAYOUT_INTERNAL 1 /* GEMM-native parity-folded layout (sph_sht_coeffs_elems) */

/* DISCO filter bases */
#define SPH_BASIS_MORLET 0    /* convolution.hpp:73-76, K = 9 */
#define SPH_BASIS_ISOTROPIC 1 /* convolution.hpp:78-81, K = 1 */

typedef struct sph_sht_plan_s* sph_sht_plan;
typedef struct sph_disco_plan_s* sph_disco_plan;

/* ---- diagnostics --------------------------------------------------------------- */
const char* sph_last_error(void);
const char* sph_version(void);
/* number of kernels this process launched through the library (all plans) */
uint64_t sph_launch_count(void);
/* stream-ordered per-kernel timing: when enabled every library kernel launch is
 * bracketed by a CUDA event pair on its own stream; sph_profile_read returns CSV
 * "name,launches,total_ms,work" aggregated since the previous read. */
int sph_profile_enable(int on);
int sph_profile_read(char* csv, size_t cap);

/* ---- grids (grid.hpp:69-128), host fp64 ---------------------------------------- */
int sph_grid(int kind, int64_t nlat, int64_t nlon, double* colatitudes, double* quad_weights);

/* ---- SHT (harmonics.hpp) --------------------------------------------------------- */
/* Replaces the per-call table builds of sht_forward/sht_inverse
 * (harmonics.hpp:159-162, :202-205): grid, Phat tables (harmonics.hpp:59-117) are
 * built once on the host in fp64, parity-folded, split hi/lo and uploaded. */
int sph_sht_plan_create(int kind, int64_t nlat, int64_t nlon, int64_t lmax, int64_t mmax,
                        int flags, sph_sht_plan* plan);
int sph_sht_plan_destroy(sph_sht_plan plan);
/* element counts (floats) of a coefficient buffer for F fields in `layout` */
int64_t sph_sht_coeffs_elems(sph_sht_plan plan, int64_t F, int layout);
/* bytes of caller workspace needed by forward/inverse for F fields */
int64_t sph_sht_workspace_bytes(sph_sht_plan plan, int64_t F);

/* sphere::sht_forward (harmonics.hpp:126 / :159 / :164; equiangular arithmetic of
 * distsim.hpp:413-459).  x: fields [F][nlat][nlon]; coeffs: F fields in `layout`.
 * workspace: >= sph_sht_workspace_bytes(plan, F) bytes of device memory, or NULL to use
 * a plan-owned buffer (then calls on the same plan must be serialised). */
int sph_sht_forward(sph_sht_plan plan, const float* x, int64_t F, float* coeffs, int layout,
                    void* workspace, void* stream);
/* sphere::sht_inverse (harmonics.hpp:173 / :202) */
int sph_sht_inverse(sph_sht_plan plan, const float* coeffs, int64_t F, int layout, float* y,
                    void* workspace, void* stream);
/* sht_inverse(sht_forward(x)) for HOST buffers (pageable or pinned): the F fields are
 * streamed through the device in chunks with H2D / compute / D2H overlapped on
 * internal streams.  Blocks until y_host is written. */
int sph_sht_roundtrip_host(sph_sht_plan plan, const float* x_host, int64_t F, float* y_host,
                           int64_t chunk_fields);

/* Stage entry points used by the distributed (pencil) SHT, distsim.hpp:404-463.
 * fft stage: rings [F][h_count][nlon] -> bins [F][h_count][mmax] complex64, scaled
 *   by 2*pi/nlon (distsim.hpp:413-430).
 * legendre stage: bins [F][nlat][m_count] complex64 for global orders
 *   m0..m0+m_count-1 -> coeffs [F][lmax][m_count] complex64 (distsim.hpp:437-459). */
int sph_sht_fft_stage(sph_sht_plan plan, const float* rings, int64_t F, int64_t h_count,
                      float* bins, void* stream);
int sph_sht_legendre_stage(sph_sht_plan plan, const float* bins, int64_t F, int64_t m0,
                           int64_t m_count, float* coeffs, void* workspace, void* stream);
int64_t sph_sht_stage_workspace_bytes(sph_sht_plan plan, int64_t F, int64_t m_count);

/* ---- DISCO (convolution.hpp) --------------------------------------------------- */
/* assemble_disco (convolution.hpp:141-177) on the host in fp64, then the device
 * tables.  Errors as the reference: longitudes not a uniform subset (:143-145) and empty
 * support rows (:172-174) -> SPH_ERR_INVALID_ARGUMENT. */
int sph_disco_plan_create(int in_kind, int64_t in_nlat, int64_t in_nlon, int out_kind,
                          int64_t out_nlat, int64_t out_nlon, int basis, double theta_cutoff,
                          int flags, sph_disco_plan* plan);
int sph_disco_plan_destroy(sph_disco_plan plan);
/* K (real basis functions), stride, total entries per basis function */
int sph_disco_plan_info(sph_disco_plan plan, int64_t* n_basis, int64_t* stride,
                        int64_t* nnz_per_basis);
int64_t sph_disco_workspace_bytes(sph_disco_plan plan, int64_t B, int64_t c_in, int64_t c_out);
/* disco_apply (convolution.hpp:181-220): x [B][c_in][in_nlat][in_nlon],
 * mix [c_out][c_in][K], y [B][c_out][out_nlat][out_nlon]. */
int sph_disco_apply(sph_disco_plan plan, const float* x, const float* mix, int64_t B,
                    int64_t c_in, int64_t c_out, float* y, void* workspace, void* stream);

/* disco_transpose_apply (convolution.hpp:226-266): the adjoint of sph_disco_apply under
 * the grids' quadrature inner products (entries re-weighted with the output grid's weight,
 * :251).  v [B][c_out][out_nlat][out_nlon] on the OUTPUT grid, mix [c_out][c_in][K] (the
 * forward's mix tensor) -> y [B][c_in][in_nlat][in_nlon] on the input grid.  The
 * transposed filter tables are built on the first call. */
int64_t sph_disco_transpose_workspace_bytes(sph_disco_plan plan, int64_t B, int64_t c_in,
                                            int64_t c_out);
int sph_disco_transpose_apply(sph_disco_plan plan, const float* v, const float* mix, int64_t B,
                              int64_t c_in, int64_t c_out, float* y, void* workspace, void* stream);

/* Latitude-shard form used by the distributed DISCO (distsim.hpp:468-547 with a
 * latitude halo instead of the reduce-scatter of K-expanded partials): output rows
 * [h_out0, h_out0+n_out) from the input rows [h_in0, h_in0+n_in) given in
 * x [B][c_in][n_in][in_nlon]; y [B][c_out][n_out][out_nlon].  sph_disco_input_rows
 * returns the input row range (filter support band) those output rows need. */
int sph_disco_input_rows(sph_disco_plan plan, int64_t h_out0, int64_t n_out, int64_t* h_in0,
                         int64_t* n_in);
int64_t sph_disco_rows_workspace_bytes(sph_disco_plan plan, int64_t B, int64_t c_in, int64_t c_out,
                                       int64_t n_in, int64_t n_out);
int sph_disco_apply_rows(sph_disco_plan plan, const float* x, int64_t h_in0, int64_t n_in,
                         int64_t h_out0, int64_t n_out, const float* mix, int64_t B, int64_t c_in,
                         int64_t c_out, float* y, void* workspace, void* stream);

/* ---- grid-to-grid resampling (resample.hpp:20-114) ------------------------------ */
/* bilinear_resample with pole extension.  Grids are given by their colatitudes (host
 * fp64, increasing, as GridSpec::colatitudes) and longitude counts (longitudes are
 * 2*pi*j/nlon for every reference grid).  x [C][in_nlat][in_nlon] -> y [C][out_nlat][out_nlon]
 * (C = batch x channels fields). */
typedef struct sph_resample_plan_st* sph_resample_plan;
int sph_resample_plan_create(const double* in_colat, int64_t in_nlat, int64_t in_nlon,
                             const double* out_colat, int64_t out_nlat, int64_t out_nlon,
                             sph_resample_plan* plan);
int sph_resample_plan_destroy(sph_resample_plan plan);
int64_t sph_resample_workspace_bytes(sph_resample_plan plan, int64_t C);
int sph_bilinear_resample(sph_resample_plan plan, const float* x, int64_t C, float* y, void* workspace,
                          void* stream);

/* ---- fused decoder (model.hpp:372-394, decode_preclamp per channel group) -------- */
/* y [B][c_out][out_nlat][out_nlon] = disco_apply(dec_op, bilinear_resample(latent, out_grid), mix)
 * for latent [B][c_in][latent_nlat][latent_nlon] (latent colatitudes as in
 * sph_resample_plan_create).  `disco` is the decoder's out_grid -> out_grid operator and
 * must outlive the decoder plan.  When out_nlon is an integer multiple of latent_nlon the
 * upsampling is applied to the latent's ring spectra inside the convolution (the
 * upsampled field is never materialized); otherwise the two stages run back to back. */
typedef struct sph_decoder_plan_st* sph_decoder_plan;
int sph_decoder_plan_create(sph_disco_plan disco, const double* latent_colat, int64_t latent_nlat,
                            int64_t latent_nlon, sph_decoder_plan* plan);
int sph_decoder_plan_destroy(sph_decoder_plan plan);
int64_t sph_decoder_workspace_bytes(sph_decoder_plan plan, int64_t B, int64_t c_in, int64_t c_out);
int sph_decoder_apply(sph_decoder_plan plan, const float* latent, const float* mix, int64_t B,
                      int64_t c_in, int64_t c_out, float* y, void* workspace, void* stream);

/* ---- SHT consumers (metrics.hpp:300-314, loss.hpp:37-81) ---------------------------- */
/* Reductions over sph_sht_forward's dense output [F][lmax][mmax] complex64:
 * angular PSD psd[f][l] = |c(l,0)|^2 + 2 sum_{m=1..min(l,mmax-1)} |c(l,m)|^2, and the
 * spectral CRPS loss out[c] = sum_{1<=l<=lmax_sum, m<=min(l,mmax-1)} (m ? 2 : 1) *
 * (CRPS(Re) + CRPS(Im)) over E ensemble members (ens [E][C][lmax][mmax], obs [C][lmax][mmax];
 * variant 0 cdf, 1 spread_skill, 2 fair; out is fp64 [C]). */
int sph_psd_from_coeffs(const float* coeffs, int64_t F, int64_t lmax, int64_t mmax, float* psd,
                        void* stream);
int sph_spectral_crps_from_coeffs(const float* ens, const float* obs, int64_t E, int64_t C, int64_t lmax,
                                  int64_t mmax, int64_t lmax_sum, int variant, double* out, void* stream);
/* dist_crps local kernel (distsim.hpp:591-618): out[c] = sum_k w[k] CRPS(f[.][c][k], o[c][k]) / (4 pi)
 * over E members; f [E][C][ns], o [C][ns], w [ns] (latitude quadrature weight per sample). */
int sph_weighted_crps(const float* f, const float* o, const float* w, int64_t E, int64_t C, int64_t ns,
                      int variant, double* out, void* stream);

/* ---- spectral convolution + block epilogue ------------------------------------ */
/* spectral_conv (convolution.hpp:286-304): Gaussian grids only (:287-288);
 * kernel [c_out][c_in][klmax]; x [B][c_in][nlat][nlon] -> y [B][c_out][nlat][nlon].
 * The plan must have lmax = min(klmax, nlat), mmax = min(lmax, nlon/2) (:291-292). */
int sph_spectral_conv(sph_sht_plan plan, const float* x, const float* kernel, int64_t B,
                      int64_t c_in, int64_t c_out, int64_t klmax, float* y, void* workspace,
                      void* stream);
int64_t sph_spectral_conv_workspace_bytes(sph_sht_plan plan, int64_t B, int64_t c_in,
                                          int64_t c_out);
/* The channel mix of spectral_conv alone (convolution.hpp:295-302) on reference-layout
 * coefficients: out(b,o,l,m) = sum_i coeffs(b,i,l,m) kernel(o,i,l) for the plan's (lmax,
 * mmax); coeffs [B][c_in][lmax][mmax] complex64 -> out [B][c_out][lmax][mmax]; kernel
 * [c_out][c_in][klmax], klmax >= lmax; any grid kind.  Workspace as sph_spectral_conv. */
int sph_spectral_mix(sph_sht_plan plan, const float* coeffs, const float* kernel, int64_t B, int64_t c_in,
                     int64_t c_out, int64_t klmax, float* out, void* workspace, void* stream);
/* block_apply epilogue (model.hpp:355-368): per point
 *   y = x + scales .* (W2 gelu(W1 gelu(conv) + b1) + b2),  gelu exact-erfc (model.hpp:42)
 * conv, x, y: [B][C][npts]; w1 [H][C], b1 [H], w2 [C][H], b2 [C], scales [C]. */
int sph_block_epilogue(const float* conv, const float* x, const float* w1, const float* b1,
                       const float* w2, const float* b2, const float* scales, int64_t B,
                       int64_t C, int64_t H, int64_t npts, float* y, void* stream);

/* ---- domain-decomposed SHT and DISCO over NCCL (distsim.hpp:45-547) --------------- */
/* The rank cube of the reference's CommGrid (distsim.hpp:45-98): sizes = (batch, ensemble,
 * polar, azimuth), azimuth fastest.  One process per GPU; rank 0 makes the NCCL unique id
 * (sph_comm_unique_id, sph_comm_id_bytes() bytes) and the caller broadcasts it.  The
 * communicator owns the NCCL world and its (polar x azimuth) plane / azimuth groups
 * (ncclCommSplit), and the TrafficLog (distsim.hpp:120-150 schema, world-summed bytes).
 * Create on the device the plans live on (the current device). */
typedef struct sph_comm_s* sph_comm;
int64_t sph_comm_id_bytes(void);
int sph_comm_unique_id(void* id);
int sph_comm_create(const void* id, int64_t world, int64_t rank, const int64_t* sizes, sph_comm* comm);
int sph_comm_destroy(sph_comm comm);
int sph_comm_coords(sph_comm comm, int64_t* coords);
int sph_comm_traffic_csv(sph_comm comm, char* csv, size_t cap);
int sph_comm_traffic_reset(sph_comm comm);

/* dist_sht_forward (distsim.hpp:404-463, Alg. 1; no grid-kind check, like the reference)
 * and its mirror, the distributed sht_inverse (harmonics.hpp:173-205; the reference has no
 * distributed inverse).  Per (batch, ensemble) plane of nh x nw ranks, rank (i, j) holds
 *   fields  x [C][H_i][W_j]               H_i / W_j canonical splits of nlat / nlon
 *   coeffs    [C][L_i][M_j] complex64     L_i / M_j canonical splits of lmax / mmax,
 *                                          zeros above the diagonal (the unshard layout)
 * sph_dist_sht_local: {h0, hn, w0, wn, l0, ln, m0, mn, c0, cn} of this rank (c0/cn: the
 * channel slice whose transforms it computes).  `sht` is a plan of the full grid (create it
 * with SPH_FLAG_ALLOW_EQUIANGULAR_FORWARD for equiangular grids) on the comm's device; it
 * must outlive the distributed plan. */
typedef struct sph_dist_sht_plan_s* sph_dist_sht_plan;
int sph_dist_sht_plan_create(sph_comm comm, sph_sht_plan sht, int64_t C, sph_dist_sht_plan* plan);
int sph_dist_sht_plan_destroy(sph_dist_sht_plan plan);
int sph_dist_sht_local(sph_dist_sht_plan plan, int64_t* info);
int64_t sph_dist_sht_workspace_bytes(sph_dist_sht_plan plan);
int sph_dist_sht_forward(sph_dist_sht_plan plan, const float* x, float* coeffs, void* workspace, void* stream);
int sph_dist_sht_inverse(sph_dist_sht_plan plan, const float* coeffs, float* y, void* workspace, void* stream);

/* dist_disco_apply (distsim.hpp:468-547, Alg. 2 with a latitude halo instead of the
 * reduce-scatter of K-expanded partial sums): x [C_in][H_i][W_j] (input grid), mix
 * [C_out][C_in][K] replicated -> y [C_out][Ho_i][Wo_j] (output grid).  sph_dist_disco_local:
 * {h0, hn, w0, wn, ho0, hon, wo0, won, cz0, czn, need0, needn}. */
typedef struct sph_dist_disco_plan_s* sph_dist_disco_plan;
int sph_dist_disco_plan_create(sph_comm comm, sph_disco_plan op, int64_t c_in, int64_t c_out,
                               sph_dist_disco_plan* plan);
int sph_dist_disco_plan_destroy(sph_dist_disco_plan plan);
int sph_dist_disco_local(sph_dist_disco_plan plan, int64_t* info);
int64_t sph_dist_disco_workspace_bytes(sph_dist_disco_plan plan);
int sph_dist_disco_apply(sph_dist_disco_plan plan, const float* x, const float* mix, float* y, void* workspace,
                         void* stream);

/* Host-only descriptions of the exchange schedules and pack/unpack boxes (no GPU or NCCL
 * needed; the CPU tests execute them over gloo).  See csrc/dist.cu for the item codes. */
int sph_dist_sht_describe(int64_t nh, int64_t nw, int64_t q, int64_t nlat, int64_t nlon, int64_t lmax,
                          int64_t mmax, int64_t C, int what, int64_t* out, int64_t cap, int64_t* n);
int sph_dist_disco_describe(int64_t nh, int64_t nw, int64_t q, int64_t hin, int64_t win, int64_t hout, int64_t wout,
                            int64_t cin, int64_t cout, const int64_t* band_lo, const int64_t* band_n, int what,
                            int64_t* out, int64_t cap, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* SPHERE_GPU_H */
