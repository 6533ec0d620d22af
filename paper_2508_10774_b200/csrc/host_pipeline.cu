// host_pipeline.cu — blade_asa_fwd_host: the whole ASA forward (mask + block-
// sparse attention, Alg. 1 P:138-156 then P:133) on HOST buffers.
//
// The units (b, h) are independent, so the call streams them
// through the GPU in chunks of `chunk_units`, with three engines busy at once:
//
//   copy-in stream   H2D of chunk c+1's Q, K, V          (PCIe host->device)
//   caller's stream  mask + attention of chunk c          (SMs)
//   copy-out stream  D2H of chunk c-1's O, LSE, kv_cnt    (PCIe device->host)
//
// Two device slots (double buffering) live in the caller's workspace; events
// order slot reuse.  The sampler is keyed by the GLOBAL unit index
// (unit_offset + first unit of the chunk, reading R-1), so the result equals
// one blade_asa_mask + blade_bsa_fwd call over all units bit for bit.
//
// The only library state is a per-device pair of non-blocking copy streams
// and a small event set, created on first use and kept for the process.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "../../include/blade_asa.h"
#include "internal.h"

namespace blade {
int validate_mask_params(int64_t BH, int32_t N, int32_t d, const blade_asa_params_t* prm);
}

namespace {

constexpr int kMaxDevices = 64;

struct DeviceEngines {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t start = nullptr, in[2] = {}, done[2] = {}, out[2] = {};
  bool ok = false;
  std::mutex call;  // one pipelined call at a time per device (events are shared)
};

DeviceEngines g_eng[kMaxDevices];
std::mutex g_init;

DeviceEngines* engines(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return nullptr;
  std::lock_guard<std::mutex> lk(g_init);
  DeviceEngines& e = g_eng[dev];
  if (e.ok) return &e;
  const unsigned ef = cudaEventDisableTiming;
  bool ok = cudaStreamCreateWithFlags(&e.h2d, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&e.d2h, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&e.start, ef) == cudaSuccess;
  for (int s = 0; s < 2 && ok; ++s)
    ok = cudaEventCreateWithFlags(&e.in[s], ef) == cudaSuccess &&
         cudaEventCreateWithFlags(&e.done[s], ef) == cudaSuccess &&
         cudaEventCreateWithFlags(&e.out[s], ef) == cudaSuccess;
  e.ok = ok;
  return ok ? &e : nullptr;
}

// Carve-up of the caller's device workspace: two slots of per-chunk tensors,
// then one blade_asa_fwd scratch (compute is serial on one stream).
struct HostWs {
  size_t q, k, v, o, lse, idx, cnt, slot, mask_ws, attn_ws, off_mask, off_attn, total;
};

HostWs host_ws_layout(int64_t C, int N, int d, int Nb, size_t mask_ws, size_t attn_ws) {
  HostWs w{};
  const size_t tok = size_t(C) * N * d * 2;
  size_t o = 0;
  w.q = o;   o = blade::align256(o + tok);
  w.k = o;   o = blade::align256(o + tok);
  w.v = o;   o = blade::align256(o + tok);
  w.o = o;   o = blade::align256(o + tok);
  w.lse = o; o = blade::align256(o + size_t(C) * N * 4);
  w.idx = o; o = blade::align256(o + size_t(C) * Nb * Nb * 4);
  w.cnt = o; o = blade::align256(o + size_t(C) * Nb * 4);
  w.slot = o;
  w.off_mask = 2 * w.slot;
  w.mask_ws = mask_ws;
  w.off_attn = blade::align256(w.off_mask + mask_ws);
  w.attn_ws = attn_ws;
  w.total = blade::align256(w.off_attn + attn_ws);
  return w;
}

int64_t auto_chunk(int64_t BH, int32_t chunk_units) {
  if (chunk_units > 0) return chunk_units < BH ? chunk_units : BH;
  const int64_t c = (BH + 15) / 16;  // >= 16 chunks' worth of overlap, >= 1 unit
  return c < 1 ? 1 : c;
}

bool sizes(int64_t BH, int32_t N, int32_t d, const blade_asa_params_t* p, int32_t chunk_units,
           HostWs* out, int64_t* C_out) {
  if (BH < 1 || N < 1 || !p || chunk_units < 0) return false;
  const int64_t C = auto_chunk(BH, chunk_units);
  const size_t fws = blade_asa_fwd_workspace_size(C, N, d, p);  // mask + attention scratch
  if (fws == 0) return false;
  const int Nb = int((int64_t(N) + p->block - 1) / p->block);
  *out = host_ws_layout(C, N, d, Nb, fws, 0);
  *C_out = C;
  return true;
}

}  // namespace

extern "C" {

size_t blade_asa_fwd_host_workspace_size(int64_t BH, int32_t N, int32_t d,
                                         const blade_asa_params_t* params,
                                         int32_t chunk_units) {
  HostWs w;
  int64_t C;
  return sizes(BH, N, d, params, chunk_units, &w, &C) ? w.total : 0;
}

blade_status_t blade_asa_fwd_host(const void* q_host, const void* k_host, const void* v_host,
                                  int64_t BH, int32_t N, int32_t d,
                                  const blade_asa_params_t* params, int32_t impl,
                                  int32_t chunk_units, void* o_host, float* lse_host,
                                  int32_t* kv_cnt_host, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  if (!q_host || !k_host || !v_host || !o_host || !params) return BLADE_ERR_INVALID_ARG;
  if (impl < BLADE_ATTN_AUTO || impl > BLADE_ATTN_TCGEN05_TRIPLE) return BLADE_ERR_INVALID_ARG;
  HostWs w;
  int64_t C;
  if (!sizes(BH, N, d, params, chunk_units, &w, &C)) {
    // distinguish bad arguments from GPU limits the way the device calls do
    if (chunk_units < 0) return BLADE_ERR_INVALID_ARG;
    const int st = blade::validate_mask_params(BH, N, d, params);
    return st != BLADE_OK ? blade_status_t(st) : BLADE_ERR_UNSUPPORTED;
  }
  if (!workspace || workspace_bytes < w.total || (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return BLADE_ERR_WORKSPACE;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return BLADE_ERR_CUDA;
  DeviceEngines* eng = engines(dev);
  if (!eng) return BLADE_ERR_CUDA;
  std::lock_guard<std::mutex> lk(eng->call);

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  const int Nb = int((int64_t(N) + params->block - 1) / params->block);
  const size_t row_tok = size_t(N) * d * 2;  // bytes of one unit of Q/K/V/O
  auto fail = [](cudaError_t e) { return e == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA; };
#define BLADE_TRY(x)                                   \
  do {                                                 \
    cudaError_t e_ = (x);                              \
    if (e_ != cudaSuccess) return fail(e_);            \
  } while (0)

  // everything already on the caller's stream (e.g. users of the workspace)
  // happens before the first copy
  BLADE_TRY(cudaEventRecord(eng->start, s));
  BLADE_TRY(cudaStreamWaitEvent(eng->h2d, eng->start, 0));
  BLADE_TRY(cudaStreamWaitEvent(eng->d2h, eng->start, 0));

  const int64_t nchunks = (BH + C - 1) / C;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int sl = int(c & 1);
    const int64_t u0 = c * C;
    const int64_t cu = (u0 + C <= BH) ? C : BH - u0;
    char* base = ws + sl * w.slot;
    void *dq = base + w.q, *dk = base + w.k, *dv = base + w.v, *dO = base + w.o;
    float* dlse = reinterpret_cast<float*>(base + w.lse);
    int32_t* didx = reinterpret_cast<int32_t*>(base + w.idx);
    int32_t* dcnt = reinterpret_cast<int32_t*>(base + w.cnt);
    const size_t nb = size_t(cu) * row_tok, off = size_t(u0) * row_tok;

    // copy-in: the slot's inputs are free once chunk c-2's compute is done
    BLADE_TRY(cudaStreamWaitEvent(eng->h2d, eng->done[sl], 0));
    BLADE_TRY(cudaMemcpyAsync(dq, static_cast<const char*>(q_host) + off, nb,
                              cudaMemcpyHostToDevice, eng->h2d));
    BLADE_TRY(cudaMemcpyAsync(dk, static_cast<const char*>(k_host) + off, nb,
                              cudaMemcpyHostToDevice, eng->h2d));
    BLADE_TRY(cudaMemcpyAsync(dv, static_cast<const char*>(v_host) + off, nb,
                              cudaMemcpyHostToDevice, eng->h2d));
    BLADE_TRY(cudaEventRecord(eng->in[sl], eng->h2d));

    // compute on the caller's stream: after the inputs landed and after chunk
    // c-2's outputs left the slot
    BLADE_TRY(cudaStreamWaitEvent(s, eng->in[sl], 0));
    BLADE_TRY(cudaStreamWaitEvent(s, eng->out[sl], 0));
    blade_asa_params_t pc = *params;
    pc.unit_offset = params->unit_offset + u0;
    // mask + attention as one call (the attention a programmatic dependent of
    // the mask's refinement); its scratch is the contiguous mask + attention
    // region of the workspace (same layout blade_asa_fwd expects)
    blade_status_t st = blade_asa_fwd(dq, dk, dv, cu, N, d, &pc, impl, didx, dcnt, dO,
                                      lse_host ? dlse : nullptr, ws + w.off_mask,
                                      w.total - w.off_mask, s);
    if (st != BLADE_OK) return st;
    BLADE_TRY(cudaEventRecord(eng->done[sl], s));

    // copy-out
    BLADE_TRY(cudaStreamWaitEvent(eng->d2h, eng->done[sl], 0));
    BLADE_TRY(cudaMemcpyAsync(static_cast<char*>(o_host) + off, dO, nb, cudaMemcpyDeviceToHost,
                              eng->d2h));
    if (lse_host)
      BLADE_TRY(cudaMemcpyAsync(lse_host + u0 * N, dlse, size_t(cu) * N * 4,
                                cudaMemcpyDeviceToHost, eng->d2h));
    if (kv_cnt_host)
      BLADE_TRY(cudaMemcpyAsync(kv_cnt_host + u0 * Nb, dcnt, size_t(cu) * Nb * 4,
                                cudaMemcpyDeviceToHost, eng->d2h));
    BLADE_TRY(cudaEventRecord(eng->out[sl], eng->d2h));
  }
  // the caller's stream completes only after every output reached the host
  for (int sl = 0; sl < 2 && sl < nchunks; ++sl) BLADE_TRY(cudaStreamWaitEvent(s, eng->out[sl], 0));
#undef BLADE_TRY
  return BLADE_OK;
}

}  // extern "C"
