// internal.h — launcher declarations and workspace layout shared by the
// C-ABI front end (abi.cu) and the kernel translation units.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace blade {

struct MaskProblem {
  int64_t BH;
  int N, d, b, kk, Nb;
  double tau;
  int lo, hi;
  float scale;
  uint64_t seed;
  int mode, share_qk;
  int64_t unit_offset;
  double guard;
  int neg_flagged;  // blade_asa_fwd: refined rows' kv_cnt provisional (-1 - m) until K-mask.4
  int32_t* lpt_order;  // blade_asa_fwd: LPT order of the attention CTAs, written before K-mask.4
  int lpt_pairs;       // order over pairs of query blocks (two-block kernel)
  int* attn_work;      // blade_asa_fwd: the persistent attention's item counter, zeroed by K-mask.1
};

// Workspace carve-up for blade_asa_mask (all offsets 256-byte aligned).
struct MaskWorkspace {
  size_t off_qs, off_ks, off_pimp, off_counters, off_flags, off_done, off_r64,
      off_mpart, off_lpart, total;
  int nchunks;  // refine key chunks of 128 sampled keys
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// K-mask.2 (probe2.cu, tcgen05): k in {16, 32, 64, 128}, N_b <= 512.
bool probe2_supported(int d, int kk, int Nb, int64_t BH, int N);

inline MaskWorkspace mask_workspace_layout(const MaskProblem& p) {
  MaskWorkspace w{};
  const size_t rows = size_t(p.BH) * p.Nb;            // (unit, q-block) rows
  const size_t nk = size_t(p.Nb) * p.kk;              // padded sampled rows / unit
  const size_t ck = 128;  // sampled keys per refine work item (RF_CK)
  w.nchunks = int((nk + ck - 1) / ck);
  const size_t gath = size_t(p.BH) * nk * p.d * 2;  // gathered sampled rows
  size_t o = 0;
  w.off_qs = o;       o = align256(o + gath);
  w.off_ks = o;       o = align256(o + gath);
  w.off_pimp = o;     o = align256(o + rows * p.Nb * 4);
  w.off_counters = o; o = align256(o + 64);  // [0] refine queue length
  w.off_flags = o;    o = align256(o + rows * 4);
  w.off_done = o;     o = align256(o + rows * 4);
  w.off_r64 = o;      o = align256(o + rows * p.kk * p.Nb * 8);
  w.off_mpart = o;    o = align256(o + rows * w.nchunks * p.kk * 8);
  w.off_lpart = o;    o = align256(o + rows * w.nchunks * p.kk * 8);
  w.total = o;
  return w;
}

cudaError_t launch_mask(const MaskProblem& p, const void* q, const void* k, uint8_t* mask,
                        int32_t* kv_idx, int32_t* kv_cnt, float* p_imp_out,
                        int32_t* sample_idx, int32_t* n_refined, char* ws,
                        cudaStream_t stream);

cudaError_t launch_probe2(int64_t BH, int N, int Nb, int b, int kk, int d, float scale,
                          const void* qs, const void* ks, float* pimp, cudaStream_t stream);
// Attention implementations compiled into this library: AUTO / TCGEN05_PAIR
// (attn_tc2.cu) and TCGEN05 (attn_tc.cu) always; the mma.sync and
// three-S-buffer kernels only into -DBLADE_WITH_BASELINES builds.
inline bool impl_built(int impl) {
#ifdef BLADE_WITH_BASELINES
  return impl >= 0 && impl <= 4;
#else
  return impl == 0 || impl == 1 || impl == 3;
#endif
}

struct AttnProblem {
  int64_t BH;
  int N, d, b, Nb;
  float scale;
};

cudaError_t launch_attn_mma(const AttnProblem& p, const void* q, const void* k,
                            const void* v, const int32_t* kv_idx, const int32_t* kv_cnt,
                            void* o, float* lse, cudaStream_t stream);

// ASA_GT global tokens: pooled K/V [BH, Ng, d] bf16 and the window n.
struct GtProblem {
  const void* kg;
  const void* vg;
  int Ng, window;
};

// Returns cudaErrorNotSupported when the tcgen05 path is not available.
// pdl: launched as a programmatic dependent of the refine kernel (blade_asa_fwd);
// CTAs whose kv_cnt is negative (provisional) wait for it to complete.
cudaError_t launch_attn_tc(const AttnProblem& p, const void* q, const void* k,
                           const void* v, const int32_t* kv_idx, const int32_t* kv_cnt,
                           void* o, float* lse, char* ws, size_t ws_bytes,
                           cudaStream_t stream, const GtProblem* gt = nullptr, bool pdl = false,
                           const int32_t* order = nullptr);

// Two query blocks per CTA (ping-pong softmax warpgroups), attn_tc2.cu.
cudaError_t launch_attn_tc2(const AttnProblem& p, const void* q, const void* k, const void* v,
                            const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                            cudaStream_t stream, const GtProblem* gt = nullptr, bool pdl = false,
                            const int32_t* order = nullptr);

// The pair kernel as a persistent kernel (attn_tc2p.cu): one CTA per SM
// claims (unit, pair) items from the counter `work` (an int of the attention
// workspace, zeroed on the stream by the launcher); BLADE_ATTN_AUTO uses it.
cudaError_t launch_attn_tc2p(const AttnProblem& p, const void* q, const void* k, const void* v,
                             const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                             int* work, bool work_zeroed, cudaStream_t stream,
                             const GtProblem* gt = nullptr, bool pdl = false,
                             const int32_t* order = nullptr);
// work_zeroed: K-mask.1 of the same call zeroed the counter (blade_asa_fwd; a
// memset here would sit between K-mask.4 and the attention and break the
// programmatic dependent launch), else it is zeroed here.
inline cudaError_t launch_attn_auto(const AttnProblem& p, const void* q, const void* k,
                                    const void* v, const int32_t* kv_idx, const int32_t* kv_cnt,
                                    void* o, float* lse, void* workspace, cudaStream_t stream,
                                    const GtProblem* gt = nullptr, bool pdl = false,
                                    const int32_t* order = nullptr, bool work_zeroed = false) {
#ifdef BLADE_ATTN2P_OFF  // A/B: the non-persistent pair kernel
  (void)workspace;
  (void)work_zeroed;
  return launch_attn_tc2(p, q, k, v, kv_idx, kv_cnt, o, lse, stream, gt, pdl, order);
#else
  return launch_attn_tc2p(p, q, k, v, kv_idx, kv_cnt, o, lse, static_cast<int*>(workspace),
                          work_zeroed, stream, gt, pdl, order);
#endif
}

// Longest-processing-time order of the attention CTAs (one query block, or a
// pair of blocks when pairs != 0) by kept-block count, descending; counts may
// be provisional (negative: -1 - m).  order: [BH * ceil(Nb / (pairs ? 2 : 1))].
cudaError_t launch_lpt_order(const int32_t* kv_cnt, int64_t BH, int Nb, int d, int pairs,
                             int32_t* order, cudaStream_t stream);

// Block-sparse attention backward (attn_bwd.cu): workspace = D_r (fp32
// [BH, N]) + transposed lists q_idx [BH, N_b, N_b] + q_cnt [BH, N_b].
struct BwdWorkspace {
  size_t off_d, off_qidx, off_qcnt, total;
};
inline BwdWorkspace bwd_workspace_layout(const AttnProblem& p) {
  BwdWorkspace w{};
  size_t o = 0;
  w.off_d = o;    o = align256(o + size_t(p.BH) * p.N * 4);
  w.off_qidx = o; o = align256(o + size_t(p.BH) * p.Nb * p.Nb * 4);
  w.off_qcnt = o; o = align256(o + size_t(p.BH) * p.Nb * 4);
  w.total = o;
  return w;
}
cudaError_t launch_attn_bwd(const AttnProblem& p, const void* q, const void* k, const void* v,
                            const void* o, const float* lse, const void* dout,
                            const int32_t* kv_idx, const int32_t* kv_cnt, void* dq, void* dk,
                            void* dv, char* ws, cudaStream_t stream);

// ASA_GT backward (attn_bwd.cu): the plain backward's workspace, then the
// global tokens' fp32 partial sums part [2][splits][BH][Ngp][d] (the query
// blocks split so the grid covers the SMs) and their reduction gsum [2][BH][Ng][d].
struct GtBwdWorkspace {
  int splits, Ngp;
  size_t off_part, off_gsum, total;
};
inline GtBwdWorkspace gt_bwd_workspace_layout(const AttnProblem& p, int Ng) {
  GtBwdWorkspace w{};
  w.Ngp = (Ng + 127) / 128 * 128;  // whole 128-row tiles (tcgen05 kernel; 64 for mma.sync)
  const int64_t ctas = p.BH * (w.Ngp / 128);  // one CTA per SM: about four waves
  int s = int((4 * 148 + ctas - 1) / ctas);
  s = s < 1 ? 1 : (s > 64 ? 64 : s);
  w.splits = s > p.Nb ? p.Nb : s;
  size_t o = bwd_workspace_layout(p).total;
  w.off_part = o; o = align256(o + 2 * size_t(w.splits) * p.BH * w.Ngp * p.d * 4);
  w.off_gsum = o; o = align256(o + 2 * size_t(p.BH) * Ng * p.d * 4);
  w.total = o;
  return w;
}
cudaError_t launch_attn_gt_bwd(const AttnProblem& p, const GtProblem& gp, const void* q,
                               const void* k, const void* v, const void* o, const float* lse,
                               const void* dout, const int32_t* kv_idx, const int32_t* kv_cnt,
                               void* dq, void* dk, void* dv, char* ws, cudaStream_t stream);

// dQ of the backward on tcgen05 (attn_bwd_tc.cu); cudaErrorNotSupported if the
// tensor maps cannot be built.
// gt != nullptr: dK/dV of the global tokens (K_g/V_g tiles against every
// query block, `splits` query ranges) into fp32 partials `part` laid out as
// GtBwdWorkspace; dQ with the global-token tiles appended to every list.
cudaError_t launch_bwd_dkdv_tc(const AttnProblem& p, const void* q, const void* k, const void* v,
                               const float* lse, const void* dout, const float* Dv,
                               const int32_t* q_idx, const int32_t* q_cnt, void* dk, void* dv,
                               cudaStream_t stream, const GtProblem* gt = nullptr,
                               float* part = nullptr, int splits = 1);
cudaError_t launch_bwd_dq_tc(const AttnProblem& p, const void* q, const void* k, const void* v,
                             const float* lse, const void* dout, const float* Dv,
                             const int32_t* kv_idx, const int32_t* kv_cnt, void* dq,
                             cudaStream_t stream, const GtProblem* gt = nullptr);

// One query block per CTA, three S buffers in TMEM (attn_tc3.cu).
cudaError_t launch_attn_tc3(const AttnProblem& p, const void* q, const void* k, const void* v,
                            const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                            cudaStream_t stream, const GtProblem* gt = nullptr);

// MeanPool_n of K and V, fp32 accumulation, bf16 round-to-nearest.
cudaError_t launch_gt_pool(const void* k, const void* v, int64_t BH, int N, int d, int window,
                           void* kg, void* vg, cudaStream_t stream);
size_t attn_tc_workspace(const AttnProblem& p);

}  // namespace blade
