/*
 * blade_asa.h — C ABI of the B200-native ASA forward (BLADE, arXiv 2508.10774).
 *
 * Two calls make up the hot path of Adaptive Block-Sparse Attention (ASA):
 *
 *   blade_asa_mask  Alg. 1 of the paper with Alg. 2/3
 *                    as the definition of the block importance
 *                   P_imp: block partition (l.2), random sampling of k tokens
 *                   per block of Q and K (l.3), the sampled attention
 *                   softmax(Q_s K_s^T * scale) (l.4), k x k max-pooling to
 *                   P_imp (l.5), row normalisation, descending sort,
 *                   cumulative-mass cut at tau and clamping (l.7-9), and the
 *                   binary mask (l.10), compacted to per-query-block lists of
 *                   kept key blocks.
 *   blade_bsa_fwd   block-sparse flash-attention forward ("Standard
 *                   ASA: the generated binary sparse mask M is directly
 *                   integrated with a block-sparse attention kernel") over
 *                   those lists, producing O and the log-sum-exp LSE.
 *
 * Conventions shared by every entry point
 *   - Tensors are caller-owned DEVICE memory, contiguous, layout [BH, N, d]
 *     with BH = B*H flattened (unit u = b*H + h), so a contiguous range of
 *     units is a contiguous slice.  Q, K, V, O are bf16 (raw 16-bit words).
 *   - Nothing is allocated or freed by the library.  Scratch comes from the
 *     caller's `workspace` (device memory, >= the size the matching
 *     *_workspace_size() returns, 256-byte aligned).  The library writes it
 *     (e.g. the persistent attention's item counter), so one workspace must
 *     not serve two calls that can run concurrently (different streams).
 *   - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *     stream).  Calls never synchronise the host.
 *   - Arguments are validated synchronously before anything is enqueued; a
 *     non-OK status means nothing was launched.  Launch failures return
 *     BLADE_ERR_CUDA (cudaGetLastError).  No C++ exception crosses the ABI.
 *   - Non-finite inputs give undefined (but memory-safe) outputs.
 *   - The device entry points are stateless and re-entrant (the host-buffer
 *     entry point keeps per-device copy streams, see below).
 *   - GPU limits: block (b) == 128; d in {64, 128}; samples (k) in
 *     {16, 32, 64, 128}; N >= 1; N_b = ceil(N/b) <= 512.  Other values give
 *     BLADE_ERR_UNSUPPORTED.
 */
#ifndef BLADE_ASA_H_
#define BLADE_ASA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BLADE_OK = 0,
  BLADE_ERR_INVALID_ARG = 1,   /* NULL / misaligned pointer, bad size or parameter */
  BLADE_ERR_UNSUPPORTED = 2,   /* valid per the paper but outside the GPU limits above */
  BLADE_ERR_WORKSPACE = 3,     /* workspace NULL or smaller than *_workspace_size() */
  BLADE_ERR_CUDA = 4           /* a CUDA launch or runtime call failed */
} blade_status_t;

/* Mask-generation parameters.  Field readings: DESIGN.md §Readings. */
typedef struct {
  int32_t  block;        /* b, query and key block size ("b=128"); GPU: 128       */
  int32_t  samples;      /* k, tokens sampled per block ("k=16"); 1 <= k <= b     */
  float    tau;          /* cumulative-mass threshold, 0 < tau <= 1       */
  int32_t  keep_min;     /* lo: min kept key blocks per query block, >= 1 (P:151 clamp) */
  int32_t  keep_max;     /* hi: max kept, >= lo; clipped to N_b.  lo == hi: top-k mode  */
  float    scale;        /* softmax scale, normally (float)(1/sqrt(d))           */
  uint64_t seed;         /* sampler seed (reading R-1)                                   */
  int32_t  sample_mode;  /* 0 hash-random (default, R-1), 1 strided, 2 caller-supplied  */
  int32_t  share_qk;     /* 0: independent Q and K samples; 1: K reuses Q's offsets     */
  int64_t  unit_offset;  /* global index of this call's first unit (sharding, R-1)      */
  float    refine_guard; /* relative decision margin below which a row is recomputed in
                            fp64 (reading R-14); <= 0 selects the default 1e-5          */
  int32_t  reserved;     /* must be 0                                                    */
} blade_asa_params_t;

/* Bytes of scratch blade_asa_mask needs for this problem (0 on bad args). */
size_t blade_asa_mask_workspace_size(int64_t BH, int32_t N, int32_t d,
                                     const blade_asa_params_t* params);

/*
 * blade_asa_mask — Alg. 1 l.2-10 for every unit.
 *   q, k        [BH, N, d] bf16 device, 16-byte aligned (required).
 *   mask        [BH, N_b, N_b] uint8 0/1 out (optional, may be NULL).
 *   kv_idx      [BH, N_b, N_b] int32 out (required): row i lists the kept key
 *               blocks of query block i in ascending order, tail = -1.
 *   kv_cnt      [BH, N_b] int32 out (required): m of row i, in [lo, hi].
 *   p_imp       [BH, N_b, N_b] fp32 out (optional): raw max-pooled P_imp of
 *               Alg. 1 l.5 (before the l.7 normalisation).  Rows decided in
 *               fp64 (refined) hold that fp64 value rounded to fp32.
 *   sample_idx  [BH, 2, N_b, k] int32 (optional): in-block offsets of the
 *               sampled Q ([:,0]) and K ([:,1]) rows, ascending, -1 padded.
 *               OUTPUT for sample_mode 0/1; INPUT (required) for mode 2:
 *               block i's first k_i = min(k, valid_i) entries must be
 *               distinct offsets in [0, valid_i) (not checked; other values
 *               give undefined results, possibly out-of-range reads).
 *   n_refined   device int32 scalar out (optional): rows recomputed in fp64.
 * Errors: INVALID_ARG (NULL q/k/kv_idx/kv_cnt, N < 1, BH < 1, tau out of
 * (0, 1], lo < 1, hi < lo, k < 1 or k > b, reserved != 0, mode 2 without
 * sample_idx), UNSUPPORTED (GPU limits: d not 64/128, b != 128, k not in
 * {16, 32, 64, 128}, N_b > 512, BH > 65535), WORKSPACE, CUDA.
 */
blade_status_t blade_asa_mask(const void* q, const void* k, int64_t BH, int32_t N,
                              int32_t d, const blade_asa_params_t* params,
                              uint8_t* mask, int32_t* kv_idx, int32_t* kv_cnt,
                              float* p_imp, int32_t* sample_idx, int32_t* n_refined,
                              void* workspace, size_t workspace_bytes,
                              void* stream);

/* Bytes of scratch blade_bsa_fwd needs (0 on bad args). */
size_t blade_bsa_fwd_workspace_size(int64_t BH, int32_t N, int32_t d, int32_t block);

/* Attention implementations (the `impl` argument of blade_bsa_fwd). */
#define BLADE_ATTN_AUTO 0      /* fastest measured, d = 64 and 128: the pair schedule of
                                  TCGEN05_PAIR as a persistent kernel (one CTA per SM
                                  claiming (unit, pair of query blocks) items)          */
#define BLADE_ATTN_TCGEN05 1   /* sm_100a tcgen05 + TMEM + TMA warp-specialised kernel */
#define BLADE_ATTN_MMA_SYNC 2  /* legacy mma.sync baseline (BLADE_WITH_BASELINES builds)  */
#define BLADE_ATTN_TCGEN05_PAIR 3 /* tcgen05 kernel with two query blocks per CTA (ping-pong) */
#define BLADE_ATTN_TCGEN05_TRIPLE 4 /* one query block, three S buffers (baseline builds) */

/*
 * blade_bsa_fwd — block-sparse attention over kept blocks.
 *   For each query row r of query block i and T = union of [j*b, min(j*b+b, N))
 *   over j in kv_idx[u, i, 0:kv_cnt[u, i]]:
 *     LSE[r] = ln sum_{t in T} exp(scale * q_r . k_t)            (reading R-10)
 *     O[r]   = sum_{t in T} exp(scale * q_r . k_t - LSE[r]) * v_t
 *   q, k, v     [BH, N, d] bf16 device, 16-byte aligned.
 *   kv_idx      [BH, N_b, N_b] int32, kv_cnt [BH, N_b] int32 (e.g. from
 *               blade_asa_mask; caller-built lists must hold distinct ids in
 *               [0, N_b), 1 <= kv_cnt <= N_b; order is free).
 *   o           [BH, N, d] bf16 out; lse [BH, N] fp32 out (may be NULL).
 *   impl        BLADE_ATTN_* selector.
 * Errors: INVALID_ARG, UNSUPPORTED (GPU limits: d not 64/128, block != 128,
 * N_b > 512, BH > 65535; impl not built), WORKSPACE, CUDA.  All checks run
 * before anything is enqueued.
 */
blade_status_t blade_bsa_fwd(const void* q, const void* k, const void* v, int64_t BH,
                             int32_t N, int32_t d, int32_t block, float scale,
                             const int32_t* kv_idx, const int32_t* kv_cnt,
                             void* o, float* lse, int32_t impl,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Bytes of scratch blade_bsa_bwd needs (0 on bad args / GPU limits). */
size_t blade_bsa_bwd_workspace_size(int64_t BH, int32_t N, int32_t d, int32_t block);

/*
 * blade_bsa_bwd — gradients of blade_bsa_fwd (sparsity-aware
 * distillation trains through ASA; reading R-23: the kept-block lists are
 * constants).  With P_rt = exp(scale q_r.k_t - LSE_r) over r's kept keys:
 *   D_r = dO_r . O_r,  dV_t = sum_r P_rt dO_r,
 *   dK_t = scale sum_r P_rt (dO_r . v_t - D_r) q_r,
 *   dQ_r = scale sum_t P_rt (dO_r . v_t - D_r) k_t.
 *   q, k, v, o, dout   [BH, N, d] bf16 device (o = the forward's O), 16-B aligned.
 *   lse                [BH, N] fp32 device (the forward's LSE).
 *   kv_idx, kv_cnt     the forward's lists.
 *   dq, dk, dv         [BH, N, d] bf16 device out (every row written; key rows
 *                      no query keeps get 0).
 *   workspace          >= blade_bsa_bwd_workspace_size() (D_r and the
 *                      transposed lists).  BH <= 65535.
 * Deterministic (no atomics).  Errors: INVALID_ARG, UNSUPPORTED, WORKSPACE, CUDA.
 */
blade_status_t blade_bsa_bwd(const void* q, const void* k, const void* v, const void* o,
                             const float* lse, const void* dout, int64_t BH, int32_t N,
                             int32_t d, int32_t block, float scale, const int32_t* kv_idx,
                             const int32_t* kv_cnt, void* dq, void* dk, void* dv,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Bytes of scratch blade_asa_fwd needs (0 on bad args / GPU limits). */
size_t blade_asa_fwd_workspace_size(int64_t BH, int32_t N, int32_t d,
                                    const blade_asa_params_t* params);

/*
 * blade_asa_fwd — the whole ASA forward in one call: blade_asa_mask then
 * blade_bsa_fwd (P:138-156 then P:133), with the attention launched as a
 * programmatic dependent of the mask's last kernel (tcgen05 kernels; SURVEY
 * F4): query blocks whose selection is being recomputed in fp64 wait for it,
 * every other block starts while it runs.  Results equal the two calls.
 *   q, k, v     [BH, N, d] bf16 device; params as blade_asa_mask (sample_mode
 *               0 or 1); impl as blade_bsa_fwd.
 *   kv_idx, kv_cnt, o, lse   outputs as in the two calls (lse may be NULL);
 *               kv_cnt is final once the stream has completed.
 *   workspace   >= blade_asa_fwd_workspace_size().
 * Errors: as the two calls; UNSUPPORTED after the mask was enqueued leaves
 * kv_cnt of recomputed rows provisional (negative).
 */
blade_status_t blade_asa_fwd(const void* q, const void* k, const void* v, int64_t BH,
                             int32_t N, int32_t d, const blade_asa_params_t* params,
                             int32_t impl, int32_t* kv_idx, int32_t* kv_cnt, void* o,
                             float* lse, void* workspace, size_t workspace_bytes,
                             void* stream);

/*
 * ASA with global tokens, ASA_GT (Step 2.2 (2); readings R-18..R-20):
 * K_aug = Concat(K, MeanPool_n(K)), V_aug likewise.  Window w of the token
 * axis covers [w*n, min((w+1)*n, N)); N_g = ceil(N/n) global tokens.
 *
 * blade_gt_pool — MeanPool_n of K and V.
 *   k, v        [BH, N, d] bf16 device, 16-byte aligned.
 *   kg, vg      [BH, N_g, d] bf16 device out, 16-byte aligned: the mean of
 *               window w's n_w tokens (fp32 sum, rounded once to bf16).
 *   window      n >= 1.   BH <= 65535.
 * Errors: INVALID_ARG, UNSUPPORTED (d not in {64, 128}), CUDA.
 */
blade_status_t blade_gt_pool(const void* k, const void* v, int64_t BH, int32_t N, int32_t d,
                             int32_t window, void* kg, void* vg, void* stream);

/*
 * blade_bsa_gt_fwd — blade_bsa_fwd plus the global tokens, in one softmax:
 *   LSE[r] = ln( sum_{t in T} e^{s_t} + sum_w e^{g_w} ),
 *   O[r]   = sum_{t in T} e^{s_t - LSE[r]} v_t + sum_w e^{g_w - LSE[r]} vg_w,
 *   s_t = scale * q_r . k_t (t in the kept blocks T, as blade_bsa_fwd),
 *   g_w = scale * q_r . kg_w + ln(n_w)  for every window w (n_w = n except
 *   possibly the last window).
 *   kg, vg      [BH, N_g, d] bf16 (e.g. from blade_gt_pool), N_g = ceil(N/n).
 *   Other arguments and workspace as blade_bsa_fwd (same workspace size).
 *   impl        BLADE_ATTN_AUTO or BLADE_ATTN_TCGEN05 (MMA_SYNC: UNSUPPORTED).
 */
blade_status_t blade_bsa_gt_fwd(const void* q, const void* k, const void* v, int64_t BH,
                                int32_t N, int32_t d, int32_t block, float scale,
                                const int32_t* kv_idx, const int32_t* kv_cnt, const void* kg,
                                const void* vg, int32_t window, void* o, float* lse,
                                int32_t impl, void* workspace, size_t workspace_bytes,
                                void* stream);

/* Bytes of scratch blade_bsa_gt_bwd needs (0 on bad args / GPU limits). */
size_t blade_bsa_gt_bwd_workspace_size(int64_t BH, int32_t N, int32_t d, int32_t block,
                                       int32_t window);

/*
 * blade_bsa_gt_bwd — gradients of blade_bsa_gt_fwd with respect to q, k, v,
 * the global tokens kg = MeanPool_n(k), vg = MeanPool_n(v) included
 * (P:135 trained through P:158-161; readings R-23, R-24).  P_rt as in
 * blade_bsa_bwd with the forward's LSE (which covers the global tokens),
 * P_rw = exp(scale q_r.kg_w + ln n_w - LSE_r), dS = P (dO.v - D_r):
 *   dQ_r  = scale (sum_t dS_rt k_t + sum_w dS_rw kg_w),
 *   dK_t  = scale sum_r dS_rt q_r + dKg_{w(t)} / n_{w(t)},
 *   dV_t  = sum_r P_rt dO_r       + dVg_{w(t)} / n_{w(t)},
 *   dKg_w = scale sum_r dS_rw q_r,  dVg_w = sum_r P_rw dO_r over ALL rows r;
 * the bf16 rounding of kg, vg is passed through as the identity.
 *   kg, vg      the forward's global tokens [BH, N_g, d] bf16, N_g = ceil(N/window).
 *   o, lse      blade_bsa_gt_fwd's outputs.  Other arguments as blade_bsa_bwd.
 *   workspace   >= blade_bsa_gt_bwd_workspace_size().
 * Deterministic (no atomics).  Errors: INVALID_ARG, UNSUPPORTED, WORKSPACE, CUDA.
 */
blade_status_t blade_bsa_gt_bwd(const void* q, const void* k, const void* v, const void* kg,
                                const void* vg, int32_t window, const void* o, const float* lse,
                                const void* dout, int64_t BH, int32_t N, int32_t d,
                                int32_t block, float scale, const int32_t* kv_idx,
                                const int32_t* kv_cnt, void* dq, void* dk, void* dv,
                                void* workspace, size_t workspace_bytes, void* stream);

/*
 * blade_asa_gt_fwd — the whole ASA_GT forward in one call (P:135 with
 * P:138-156): blade_gt_pool, blade_asa_mask, then the attention over the kept
 * blocks and the global tokens launched as a programmatic dependent of the
 * mask's last kernel (as blade_asa_fwd).  Results equal blade_gt_pool +
 * blade_asa_mask + blade_bsa_gt_fwd.
 *   kg, vg      [BH, N_g, d] bf16 device OUT (N_g = ceil(N/window)): the pooled
 *               tokens, kept for blade_bsa_gt_bwd.
 *   window      n >= 1.  Other arguments as blade_asa_fwd (same workspace
 *               size, blade_asa_fwd_workspace_size); impl MMA_SYNC: UNSUPPORTED.
 */
blade_status_t blade_asa_gt_fwd(const void* q, const void* k, const void* v, int64_t BH,
                                int32_t N, int32_t d, const blade_asa_params_t* params,
                                int32_t window, int32_t impl, int32_t* kv_idx, int32_t* kv_cnt,
                                void* kg, void* vg, void* o, float* lse, void* workspace,
                                size_t workspace_bytes, void* stream);

/*
 * Locality-preserving token rearrangement ("Gilbert space-filling
 * curve to reorder the tokens before blocking"; Alg. 1 l.1; readings
 * R-21/R-22): video tokens of a t x h x w latent grid (raster order, after
 * n_text leading text tokens) are reordered frame by frame along the 2-D
 * generalised Hilbert curve of each h x w frame; text tokens stay in place.
 *
 * blade_gilbert_order — HOST function (no GPU work).
 *   perm        HOST int32 out, perm_len = n_text + t*h*w entries:
 *               perm[i] = raster index of the token placed at position i.
 * Errors: INVALID_ARG (NULL, non-positive extent, n_text < 0, wrong length).
 */
blade_status_t blade_gilbert_order(int32_t t, int32_t h, int32_t w, int32_t n_text,
                                   int32_t* perm, int64_t perm_len);

/*
 * blade_permute_tokens — DEVICE gather along the token axis of [BH, N, d]
 * bf16: inverse = 0: out[u, i, :] = x[u, perm[i], :]  (apply the order);
 *       inverse = 1: out[u, perm[i], :] = x[u, i, :]  (undo it).
 *   perm        DEVICE int32 [N], a permutation of [0, N) (not checked).
 *   x, out      distinct, 16-byte aligned; d a multiple of 8.
 * Errors: INVALID_ARG, CUDA.
 */
blade_status_t blade_permute_tokens(const void* x, int64_t BH, int32_t N, int32_t d,
                                    const int32_t* perm, int32_t inverse, void* out,
                                    void* stream);

/* Bytes of DEVICE scratch blade_asa_fwd_host needs (0 on bad args / GPU limits). */
size_t blade_asa_fwd_host_workspace_size(int64_t BH, int32_t N, int32_t d,
                                         const blade_asa_params_t* params,
                                         int32_t chunk_units);

/*
 * blade_asa_fwd_host — the whole ASA forward (blade_asa_mask, then
 * blade_bsa_fwd; P:138-156 then P:133) on HOST buffers: the units are
 * streamed through the GPU in chunks of `chunk_units` (0 = auto, about 16
 * chunks), the host->device copy of chunk c+1, the compute of chunk c and
 * the device->host copy of chunk c-1 overlapping (units are independent,
 * P:142-154).  Results equal the two device calls over all units bit for bit
 * (the sampler is keyed by params->unit_offset + global unit, reading R-1).
 *   q_host, k_host, v_host  [BH, N, d] bf16 HOST memory (page-locked for
 *               overlap; pageable memory works but copies synchronously).
 *   o_host      [BH, N, d] bf16 HOST out (required); lse_host [BH, N] fp32
 *               HOST out (optional); kv_cnt_host [BH, N_b] int32 HOST out
 *               (optional).
 *   workspace   DEVICE scratch >= blade_asa_fwd_host_workspace_size(),
 *               256-byte aligned: two chunk slots of Q/K/V/O/LSE/lists plus
 *               the mask and attention scratch.
 *   stream      compute runs on it; when it completes, every host output is
 *               written.  The host must not touch the host buffers before.
 * State: two non-blocking copy streams and a few events per device, created
 * on first use and kept for the process; concurrent calls on one device are
 * serialised while enqueuing.  Errors: as blade_asa_mask / blade_bsa_fwd.
 */
blade_status_t blade_asa_fwd_host(const void* q_host, const void* k_host, const void* v_host,
                                  int64_t BH, int32_t N, int32_t d,
                                  const blade_asa_params_t* params, int32_t impl,
                                  int32_t chunk_units, void* o_host, float* lse_host,
                                  int32_t* kv_cnt_host, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* Static, NUL-terminated description of a status code. */
const char* blade_status_string(blade_status_t status);

/* Library version as 10000*major + 100*minor + patch. */
int32_t blade_version(void);

/* 1 if attention implementation `impl` (BLADE_ATTN_*) is compiled into this
 * library, else 0.  The product build has AUTO, TCGEN05 and TCGEN05_PAIR; the
 * MMA_SYNC and TCGEN05_TRIPLE comparison kernels (and the mma.sync backward)
 * only exist in -DBLADE_WITH_BASELINES builds; elsewhere they return
 * BLADE_ERR_UNSUPPORTED. */
int32_t blade_attn_impl_built(int32_t impl);

#ifdef __cplusplus
}
#endif

#endif /* BLADE_ASA_H_ */
