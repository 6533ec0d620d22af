// abi.cu — the extern "C" boundary declared in include/blade_asa.h:
// synchronous validation, workspace accounting, and dispatch to the kernel
// launchers.  No allocation, no host synchronisation, no exceptions.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/blade_asa.h"
#include "internal.h"

namespace {

using blade::AttnProblem;
using blade::MaskProblem;

constexpr int kGpuBlock = 128;
constexpr int kMaxNb = 512;
constexpr int64_t kMaxBH = 65535;  // units ride in gridDim.y of every kernel

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

blade_status_t make_mask_problem(int64_t BH, int32_t N, int32_t d,
                                 const blade_asa_params_t* prm, MaskProblem* out) {
  if (!prm || BH < 1 || N < 1 || d < 1) return BLADE_ERR_INVALID_ARG;
  if (prm->block < 1 || prm->samples < 1 || prm->samples > prm->block) return BLADE_ERR_INVALID_ARG;
  if (!(prm->tau > 0.f && prm->tau <= 1.f)) return BLADE_ERR_INVALID_ARG;
  if (prm->keep_min < 1 || prm->keep_max < prm->keep_min) return BLADE_ERR_INVALID_ARG;
  if (prm->sample_mode < 0 || prm->sample_mode > 2 || prm->reserved != 0) return BLADE_ERR_INVALID_ARG;
  if (!(prm->scale > 0.f) || !isfinite(prm->scale)) return BLADE_ERR_INVALID_ARG;
  if (prm->unit_offset < 0) return BLADE_ERR_INVALID_ARG;
  if (prm->block != kGpuBlock || (d != 64 && d != 128)) return BLADE_ERR_UNSUPPORTED;
  if (BH > kMaxBH) return BLADE_ERR_UNSUPPORTED;
  if (prm->samples != 16 && prm->samples != 32 && prm->samples != 64 && prm->samples != 128)
    return BLADE_ERR_UNSUPPORTED;
  const int64_t Nb = (int64_t(N) + prm->block - 1) / prm->block;
  if (Nb > kMaxNb) return BLADE_ERR_UNSUPPORTED;
  MaskProblem p{};
  p.BH = BH;
  p.N = N;
  p.d = d;
  p.b = prm->block;
  p.kk = prm->samples;
  p.Nb = int(Nb);
  p.tau = double(prm->tau);  // the fp32 value, widened exactly (reading R-5)
  p.lo = int(prm->keep_min < Nb ? prm->keep_min : Nb);
  p.hi = int(prm->keep_max < Nb ? prm->keep_max : Nb);
  if (p.hi < p.lo) p.hi = p.lo;
  p.scale = prm->scale;
  p.seed = prm->seed;
  p.mode = prm->sample_mode;
  p.share_qk = prm->share_qk ? 1 : 0;
  p.unit_offset = prm->unit_offset;
  p.guard = prm->refine_guard > 0.f ? double(prm->refine_guard) : 1e-5;
  *out = p;
  return BLADE_OK;
}

}  // namespace

namespace blade {
int validate_mask_params(int64_t BH, int32_t N, int32_t d, const blade_asa_params_t* prm) {
  MaskProblem p;
  return int(make_mask_problem(BH, N, d, prm, &p));
}
}  // namespace blade

extern "C" {

size_t blade_asa_mask_workspace_size(int64_t BH, int32_t N, int32_t d,
                                     const blade_asa_params_t* params) {
  MaskProblem p;
  if (make_mask_problem(BH, N, d, params, &p) != BLADE_OK) return 0;
  return blade::mask_workspace_layout(p).total;
}

blade_status_t blade_asa_mask(const void* q, const void* k, int64_t BH, int32_t N, int32_t d,
                              const blade_asa_params_t* params, uint8_t* mask,
                              int32_t* kv_idx, int32_t* kv_cnt, float* p_imp,
                              int32_t* sample_idx, int32_t* n_refined, void* workspace,
                              size_t workspace_bytes, void* stream) {
  if (!q || !k || !kv_idx || !kv_cnt) return BLADE_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(k)) return BLADE_ERR_INVALID_ARG;
  MaskProblem p;
  blade_status_t st = make_mask_problem(BH, N, d, params, &p);
  if (st != BLADE_OK) return st;
  if (p.mode == 2 && !sample_idx) return BLADE_ERR_INVALID_ARG;
  const size_t need = blade::mask_workspace_layout(p).total;
  if (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return BLADE_ERR_WORKSPACE;
  cudaError_t e = blade::launch_mask(p, q, k, mask, kv_idx, kv_cnt, p_imp, sample_idx, n_refined,
                                     static_cast<char*>(workspace),
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA;
}

size_t blade_bsa_fwd_workspace_size(int64_t BH, int32_t N, int32_t d, int32_t block) {
  if (BH < 1 || N < 1 || block != kGpuBlock || (d != 64 && d != 128)) return 0;
  AttnProblem p{BH, N, d, block, int((N + block - 1) / block), 1.f};
  size_t a = blade::attn_tc_workspace(p);
  return a < 256 ? 256 : a;
}

blade_status_t blade_bsa_fwd(const void* q, const void* k, const void* v, int64_t BH,
                             int32_t N, int32_t d, int32_t block, float scale,
                             const int32_t* kv_idx, const int32_t* kv_cnt, void* o, float* lse,
                             int32_t impl, void* workspace, size_t workspace_bytes,
                             void* stream) {
  if (!q || !k || !v || !kv_idx || !kv_cnt || !o) return BLADE_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o)) return BLADE_ERR_INVALID_ARG;
  if (BH < 1 || N < 1 || block < 1 || !(scale > 0.f) || !isfinite(scale)) return BLADE_ERR_INVALID_ARG;
  if (impl < BLADE_ATTN_AUTO || impl > BLADE_ATTN_TCGEN05_TRIPLE) return BLADE_ERR_INVALID_ARG;
  if (block != kGpuBlock || (d != 64 && d != 128) || BH > kMaxBH) return BLADE_ERR_UNSUPPORTED;
  const int64_t Nb = (int64_t(N) + block - 1) / block;
  if (Nb > kMaxNb) return BLADE_ERR_UNSUPPORTED;
  AttnProblem p{BH, N, d, block, int(Nb), scale};
  const size_t need = blade_bsa_fwd_workspace_size(BH, N, d, block);
  if (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return BLADE_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  // AUTO: the two-blocks-per-CTA kernel, faster on B200 for both head dims
  // (interleaved A/B: Cog d = 64 1.038 vs 1.232 ms; Wan d = 128 1.170-1.180 vs
  // 1.181-1.189 ms, fused step 1.37-1.39 vs 1.40-1.43 ms)
  const bool pair = impl == BLADE_ATTN_TCGEN05_PAIR || impl == BLADE_ATTN_AUTO;
  if (!blade::impl_built(impl)) return BLADE_ERR_UNSUPPORTED;
  if (impl == BLADE_ATTN_MMA_SYNC) {
    e = blade::launch_attn_mma(p, q, k, v, kv_idx, kv_cnt, o, lse, s);
  } else if (impl == BLADE_ATTN_AUTO) {
    e = blade::launch_attn_auto(p, q, k, v, kv_idx, kv_cnt, o, lse, workspace, s);
    if (e == cudaErrorNotSupported) return BLADE_ERR_UNSUPPORTED;
  } else if (pair) {
    e = blade::launch_attn_tc2(p, q, k, v, kv_idx, kv_cnt, o, lse, s);
    if (e == cudaErrorNotSupported) return BLADE_ERR_UNSUPPORTED;
  } else if (impl == BLADE_ATTN_TCGEN05_TRIPLE) {
    e = blade::launch_attn_tc3(p, q, k, v, kv_idx, kv_cnt, o, lse, s);
    if (e == cudaErrorNotSupported) return BLADE_ERR_UNSUPPORTED;
  } else {
    e = blade::launch_attn_tc(p, q, k, v, kv_idx, kv_cnt, o, lse,
                              static_cast<char*>(workspace), workspace_bytes, s);
    if (e == cudaErrorNotSupported) return BLADE_ERR_UNSUPPORTED;
  }
  return e == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA;
}

size_t blade_asa_fwd_workspace_size(int64_t BH, int32_t N, int32_t d,
                                    const blade_asa_params_t* params) {
  const size_t m = blade_asa_mask_workspace_size(BH, N, d, params);
  const size_t a = params ? blade_bsa_fwd_workspace_size(BH, N, d, params->block) : 0;
  if (m == 0 || a == 0) return 0;
  const int64_t Nb = (int64_t(N) + params->block - 1) / params->block;
  return blade::align256(m) + blade::align256(a) + blade::align256(size_t(BH) * Nb * 4);
}

}  // extern "C"

namespace {
// blade_asa_fwd and blade_asa_gt_fwd (gt != nullptr: kg / vg are pooled here
// and attended as the global-token tiles)
blade_status_t asa_fwd_common(const void* q, const void* k, const void* v, int64_t BH, int32_t N,
                              int32_t d, const blade_asa_params_t* params, int32_t impl,
                              int32_t* kv_idx, int32_t* kv_cnt, void* o, float* lse,
                              void* workspace, size_t workspace_bytes, void* stream,
                              const blade::GtProblem* gt) {
  if (!q || !k || !v || !kv_idx || !kv_cnt || !o) return BLADE_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o)) return BLADE_ERR_INVALID_ARG;
  if (impl < BLADE_ATTN_AUTO || impl > BLADE_ATTN_TCGEN05_TRIPLE) return BLADE_ERR_INVALID_ARG;
  if (gt && impl == BLADE_ATTN_MMA_SYNC) return BLADE_ERR_UNSUPPORTED;
  if (!blade::impl_built(impl)) return BLADE_ERR_UNSUPPORTED;
  MaskProblem mp;
  blade_status_t st = make_mask_problem(BH, N, d, params, &mp);
  if (st != BLADE_OK) return st;
  if (mp.mode == 2) return BLADE_ERR_INVALID_ARG;  // supplied samples: use blade_asa_mask
  const size_t need = blade_asa_fwd_workspace_size(BH, N, d, params);
  if (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return BLADE_ERR_WORKSPACE;
  const size_t mws = blade::align256(blade::mask_workspace_layout(mp).total);
  char* ws = static_cast<char*>(workspace);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (gt) {  // MeanPool_n of K and V, independent of the mask
    e = blade::launch_gt_pool(k, v, BH, N, d, gt->window, const_cast<void*>(gt->kg),
                              const_cast<void*>(gt->vg), s);
    if (e != cudaSuccess) return BLADE_ERR_CUDA;
  }
  // programmatic dependent launch of the attention behind K-mask.4 (tcgen05
  // kernels only): rows K-mask.4 recomputes carry a provisional negative
  // count, and only their CTAs wait for it (SURVEY F4 "fused mask->attention")
  const bool pair = impl == BLADE_ATTN_TCGEN05_PAIR || impl == BLADE_ATTN_AUTO;
  const bool pdl = impl == BLADE_ATTN_AUTO || impl == BLADE_ATTN_TCGEN05 || pair;
  mp.neg_flagged = pdl ? 1 : 0;
  // LPT order of the attention CTAs when the counts vary (lo < hi); in
  // keep-ratio mode every row keeps the same number of blocks
  const size_t aws = blade::align256(blade_bsa_fwd_workspace_size(BH, N, d, mp.b));
  int32_t* order = nullptr;
  if (pdl && mp.lo < mp.hi) {
    order = reinterpret_cast<int32_t*>(ws + mws + aws);
    mp.lpt_order = order;
    mp.lpt_pairs = pair ? 1 : 0;
  }
  if (impl == BLADE_ATTN_AUTO) mp.attn_work = reinterpret_cast<int*>(ws + mws);
  e = blade::launch_mask(mp, q, k, nullptr, kv_idx, kv_cnt, nullptr, nullptr, nullptr, ws, s);
  if (e != cudaSuccess) return BLADE_ERR_CUDA;
  AttnProblem ap{BH, N, d, mp.b, mp.Nb, mp.scale};
  if (impl == BLADE_ATTN_MMA_SYNC) {
    e = blade::launch_attn_mma(ap, q, k, v, kv_idx, kv_cnt, o, lse, s);
  } else if (impl == BLADE_ATTN_TCGEN05_TRIPLE) {
    e = blade::launch_attn_tc3(ap, q, k, v, kv_idx, kv_cnt, o, lse, s, gt);
  } else if (impl == BLADE_ATTN_AUTO) {
    e = blade::launch_attn_auto(ap, q, k, v, kv_idx, kv_cnt, o, lse, ws + mws, s, gt, true,
                                order, /*work_zeroed=*/true);
  } else if (pair) {
    e = blade::launch_attn_tc2(ap, q, k, v, kv_idx, kv_cnt, o, lse, s, gt, true, order);
  } else {
    e = blade::launch_attn_tc(ap, q, k, v, kv_idx, kv_cnt, o, lse, ws + mws, aws, s, gt, true,
                              order);
  }
  if (e == cudaErrorNotSupported) return BLADE_ERR_UNSUPPORTED;
  return e == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA;
}
}  // namespace

extern "C" {

blade_status_t blade_asa_fwd(const void* q, const void* k, const void* v, int64_t BH,
                             int32_t N, int32_t d, const blade_asa_params_t* params,
                             int32_t impl, int32_t* kv_idx, int32_t* kv_cnt, void* o,
                             float* lse, void* workspace, size_t workspace_bytes,
                             void* stream) {
  return asa_fwd_common(q, k, v, BH, N, d, params, impl, kv_idx, kv_cnt, o, lse, workspace,
                        workspace_bytes, stream, nullptr);
}

blade_status_t blade_asa_gt_fwd(const void* q, const void* k, const void* v, int64_t BH,
                                int32_t N, int32_t d, const blade_asa_params_t* params,
                                int32_t window, int32_t impl, int32_t* kv_idx, int32_t* kv_cnt,
                                void* kg, void* vg, void* o, float* lse, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (!kg || !vg || !aligned16(kg) || !aligned16(vg) || window < 1) return BLADE_ERR_INVALID_ARG;
  if (BH > kMaxBH) return BLADE_ERR_UNSUPPORTED;
  if (N < 1) return BLADE_ERR_INVALID_ARG;
  const blade::GtProblem g{kg, vg, int((int64_t(N) + window - 1) / window), int(window)};
  return asa_fwd_common(q, k, v, BH, N, d, params, impl, kv_idx, kv_cnt, o, lse, workspace,
                        workspace_bytes, stream, &g);
}

blade_status_t blade_gt_pool(const void* k, const void* v, int64_t BH, int32_t N, int32_t d,
                             int32_t window, void* kg, void* vg, void* stream) {
  if (!k || !v || !kg || !vg) return BLADE_ERR_INVALID_ARG;
  if (!aligned16(k) || !aligned16(v) || !aligned16(kg) || !aligned16(vg)) return BLADE_ERR_INVALID_ARG;
  if (BH < 1 || BH > 65535 || N < 1 || window < 1) return BLADE_ERR_INVALID_ARG;
  if (d != 64 && d != 128) return BLADE_ERR_UNSUPPORTED;
  cudaError_t e = blade::launch_gt_pool(k, v, BH, N, d, window, kg, vg,
                                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA;
}

blade_status_t blade_bsa_gt_fwd(const void* q, const void* k, const void* v, int64_t BH,
                                int32_t N, int32_t d, int32_t block, float scale,
                                const int32_t* kv_idx, const int32_t* kv_cnt, const void* kg,
                                const void* vg, int32_t window, void* o, float* lse,
                                int32_t impl, void* workspace, size_t workspace_bytes,
                                void* stream) {
  if (!q || !k || !v || !kv_idx || !kv_cnt || !o || !kg || !vg) return BLADE_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(kg) ||
      !aligned16(vg))
    return BLADE_ERR_INVALID_ARG;
  if (BH < 1 || N < 1 || block < 1 || window < 1 || !(scale > 0.f) || !isfinite(scale))
    return BLADE_ERR_INVALID_ARG;
  if (impl < BLADE_ATTN_AUTO || impl > BLADE_ATTN_TCGEN05_TRIPLE) return BLADE_ERR_INVALID_ARG;
  if (block != kGpuBlock || (d != 64 && d != 128) || impl == BLADE_ATTN_MMA_SYNC ||
      BH > kMaxBH || !blade::impl_built(impl))
    return BLADE_ERR_UNSUPPORTED;
  const int64_t Nb = (int64_t(N) + block - 1) / block;
  if (Nb > kMaxNb) return BLADE_ERR_UNSUPPORTED;
  AttnProblem p{BH, N, d, block, int(Nb), scale};
  const size_t need = blade_bsa_fwd_workspace_size(BH, N, d, block);
  if (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return BLADE_ERR_WORKSPACE;
  const blade::GtProblem g{kg, vg, int((int64_t(N) + window - 1) / window), int(window)};
  cudaError_t e =
      impl == BLADE_ATTN_TCGEN05_TRIPLE
          ? blade::launch_attn_tc3(p, q, k, v, kv_idx, kv_cnt, o, lse,
                                   static_cast<cudaStream_t>(stream), &g)
      : impl == BLADE_ATTN_AUTO
          ? blade::launch_attn_auto(p, q, k, v, kv_idx, kv_cnt, o, lse, workspace,
                                    static_cast<cudaStream_t>(stream), &g)
      : impl == BLADE_ATTN_TCGEN05_PAIR
          ? blade::launch_attn_tc2(p, q, k, v, kv_idx, kv_cnt, o, lse,
                                   static_cast<cudaStream_t>(stream), &g)
          : blade::launch_attn_tc(p, q, k, v, kv_idx, kv_cnt, o, lse,
                                  static_cast<char*>(workspace), workspace_bytes,
                                  static_cast<cudaStream_t>(stream), &g);
  if (e == cudaErrorNotSupported) return BLADE_ERR_UNSUPPORTED;
  return e == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA;
}

size_t blade_bsa_bwd_workspace_size(int64_t BH, int32_t N, int32_t d, int32_t block) {
  if (BH < 1 || N < 1 || block != kGpuBlock || (d != 64 && d != 128)) return 0;
  const int64_t Nb = (int64_t(N) + block - 1) / block;
  if (Nb > kMaxNb) return 0;
  AttnProblem p{BH, N, d, block, int(Nb), 1.f};
  return blade::bwd_workspace_layout(p).total;
}

blade_status_t blade_bsa_bwd(const void* q, const void* k, const void* v, const void* o,
                             const float* lse, const void* dout, int64_t BH, int32_t N,
                             int32_t d, int32_t block, float scale, const int32_t* kv_idx,
                             const int32_t* kv_cnt, void* dq, void* dk, void* dv,
                             void* workspace, size_t workspace_bytes, void* stream) {
  if (!q || !k || !v || !o || !lse || !dout || !kv_idx || !kv_cnt || !dq || !dk || !dv)
    return BLADE_ERR_INVALID_ARG;
  for (const void* x : {q, k, v, o, dout, static_cast<const void*>(dq),
                        static_cast<const void*>(dk), static_cast<const void*>(dv)})
    if (!aligned16(x)) return BLADE_ERR_INVALID_ARG;
  if (BH < 1 || BH > 65535 || N < 1 || block < 1 || !(scale > 0.f) || !isfinite(scale))
    return BLADE_ERR_INVALID_ARG;
  if (block != kGpuBlock || (d != 64 && d != 128) || BH > kMaxBH) return BLADE_ERR_UNSUPPORTED;
  const int64_t Nb = (int64_t(N) + block - 1) / block;
  if (Nb > kMaxNb) return BLADE_ERR_UNSUPPORTED;
  AttnProblem p{BH, N, d, block, int(Nb), scale};
  const size_t need = blade::bwd_workspace_layout(p).total;
  if (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return BLADE_ERR_WORKSPACE;
  cudaError_t e = blade::launch_attn_bwd(p, q, k, v, o, lse, dout, kv_idx, kv_cnt, dq, dk, dv,
                                         static_cast<char*>(workspace),
                                         static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA;
}

size_t blade_bsa_gt_bwd_workspace_size(int64_t BH, int32_t N, int32_t d, int32_t block,
                                       int32_t window) {
  if (BH < 1 || N < 1 || window < 1 || block != kGpuBlock || (d != 64 && d != 128)) return 0;
  const int64_t Nb = (int64_t(N) + block - 1) / block;
  if (Nb > kMaxNb) return 0;
  AttnProblem p{BH, N, d, block, int(Nb), 1.f};
  return blade::gt_bwd_workspace_layout(p, int((int64_t(N) + window - 1) / window)).total;
}

blade_status_t blade_bsa_gt_bwd(const void* q, const void* k, const void* v, const void* kg,
                                const void* vg, int32_t window, const void* o, const float* lse,
                                const void* dout, int64_t BH, int32_t N, int32_t d,
                                int32_t block, float scale, const int32_t* kv_idx,
                                const int32_t* kv_cnt, void* dq, void* dk, void* dv,
                                void* workspace, size_t workspace_bytes, void* stream) {
  if (!q || !k || !v || !kg || !vg || !o || !lse || !dout || !kv_idx || !kv_cnt || !dq ||
      !dk || !dv)
    return BLADE_ERR_INVALID_ARG;
  for (const void* x : {q, k, v, kg, vg, o, dout, static_cast<const void*>(dq),
                        static_cast<const void*>(dk), static_cast<const void*>(dv)})
    if (!aligned16(x)) return BLADE_ERR_INVALID_ARG;
  if (BH < 1 || BH > 65535 || N < 1 || block < 1 || window < 1 || !(scale > 0.f) ||
      !isfinite(scale))
    return BLADE_ERR_INVALID_ARG;
  if (block != kGpuBlock || (d != 64 && d != 128) || BH > kMaxBH) return BLADE_ERR_UNSUPPORTED;
  const int64_t Nb = (int64_t(N) + block - 1) / block;
  if (Nb > kMaxNb) return BLADE_ERR_UNSUPPORTED;
  AttnProblem p{BH, N, d, block, int(Nb), scale};
  const blade::GtProblem g{kg, vg, int((int64_t(N) + window - 1) / window), int(window)};
  const size_t need = blade::gt_bwd_workspace_layout(p, g.Ng).total;
  if (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return BLADE_ERR_WORKSPACE;
  cudaError_t e = blade::launch_attn_gt_bwd(p, g, q, k, v, o, lse, dout, kv_idx, kv_cnt, dq, dk,
                                            dv, static_cast<char*>(workspace),
                                            static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA;
}

const char* blade_status_string(blade_status_t status) {
  switch (status) {
    case BLADE_OK: return "ok";
    case BLADE_ERR_INVALID_ARG: return "invalid argument";
    case BLADE_ERR_UNSUPPORTED: return "unsupported on this GPU path (see blade_asa.h limits)";
    case BLADE_ERR_WORKSPACE: return "workspace missing, misaligned or too small";
    case BLADE_ERR_CUDA: return "CUDA launch/runtime error";
  }
  return "unknown status";
}

int32_t blade_version(void) { return 200; }

int32_t blade_attn_impl_built(int32_t impl) { return blade::impl_built(impl) ? 1 : 0; }

}  // extern "C"
