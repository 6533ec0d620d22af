// gilbert.cu — locality-preserving token rearrangement (PAPER.md P:113-114
// "we employ a Gilbert space-filling curve to reorder the tokens before
// blocking"; Alg. 1 l.1).
//
//   blade_gilbert_order   HOST: the permutation.  Each h x w frame is ordered
//                         by the 2-D generalised Hilbert curve (reading R-21),
//                         frames stay in temporal order, leading text tokens
//                         keep their positions (R-22).
//   blade_permute_tokens  DEVICE: out[u, i] = x[u, perm[i]] (apply) or
//                         out[u, perm[i]] = x[u, i] (undo) for [BH, N, d] bf16;
//                         HBM-bound gather, one thread per 16-byte vector so a
//                         warp moves whole contiguous rows.
//
// Curve construction (for an arbitrary rectangle spanned by a major vector
// a and a minor vector b from corner (x, y)): a single row or column is
// walked directly; a rectangle more than 1.5x longer than wide is split into
// two halves along a; otherwise it is cut into three: a strip along b of
// half height (walked with a and b swapped), the remaining wide part, and the
// return strip walked backwards.  Halves are nudged to even lengths where
// that keeps consecutive cells adjacent.  This is the published generalised
// Hilbert ("gilbert2d") recursion of J. Cerveny (github.com/jakubcerveny/
// gilbert, BSD-2-Clause), the curve the paper names; the oracle
// (oracle/asa_oracle.py) implements the same published recursion, so the
// independent pins of both are the curve's properties (exhaustive adjacency,
// Hilbert quadrant structure, tests/test_oracle_gilbert.py), not their
// agreement.
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/blade_asa.h"

namespace {

inline int sgn(int v) { return (v > 0) - (v < 0); }

struct CurveWriter {
  int w;                  // frame width (raster stride)
  std::vector<int32_t>* out;
  void emit(int x, int y) { out->push_back(int32_t(y * w + x)); }

  void walk(int x, int y, int ax, int ay, int bx, int by) {
    const int len_a = ax + ay < 0 ? -(ax + ay) : ax + ay;
    const int len_b = bx + by < 0 ? -(bx + by) : bx + by;
    const int dax = sgn(ax), day = sgn(ay), dbx = sgn(bx), dby = sgn(by);
    if (len_b == 1) {
      for (int s = 0; s < len_a; ++s) emit(x + s * dax, y + s * day);
      return;
    }
    if (len_a == 1) {
      for (int s = 0; s < len_b; ++s) emit(x + s * dbx, y + s * dby);
      return;
    }
    int ax2 = ax / 2, ay2 = ay / 2, bx2 = bx / 2, by2 = by / 2;
    // Python-style floor division for negative components
    if (ax < 0 && ax % 2) ax2 = (ax - 1) / 2;
    if (ay < 0 && ay % 2) ay2 = (ay - 1) / 2;
    if (bx < 0 && bx % 2) bx2 = (bx - 1) / 2;
    if (by < 0 && by % 2) by2 = (by - 1) / 2;
    const int half_a = ax2 + ay2 < 0 ? -(ax2 + ay2) : ax2 + ay2;
    const int half_b = bx2 + by2 < 0 ? -(bx2 + by2) : bx2 + by2;
    if (2 * len_a > 3 * len_b) {
      if ((half_a & 1) && len_a > 2) {
        ax2 += dax;
        ay2 += day;
      }
      walk(x, y, ax2, ay2, bx, by);
      walk(x + ax2, y + ay2, ax - ax2, ay - ay2, bx, by);
    } else {
      if ((half_b & 1) && len_b > 2) {
        bx2 += dbx;
        by2 += dby;
      }
      walk(x, y, bx2, by2, ax2, ay2);
      walk(x + bx2, y + by2, ax, ay, bx - bx2, by - by2);
      walk(x + (ax - dax) + (bx2 - dbx), y + (ay - day) + (by2 - dby), -bx2, -by2, -(ax - ax2),
           -(ay - ay2));
    }
  }
};

__global__ void __launch_bounds__(256) permute_tokens_kernel(const uint4* __restrict__ x,
                                                             int64_t BH, int N, int vec_per_row,
                                                             const int32_t* __restrict__ perm,
                                                             int inverse, uint4* __restrict__ out) {
  const int64_t total = BH * N * int64_t(vec_per_row);
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < total;
       c += int64_t(gridDim.x) * blockDim.x) {
    const int v = int(c % vec_per_row);
    const int64_t row = c / vec_per_row;
    const int i = int(row % N);
    const int64_t u = row / N;
    const int p = __ldg(perm + i);
    const int64_t src = inverse ? row : u * N + p;
    const int64_t dst = inverse ? u * N + p : row;
    out[dst * vec_per_row + v] = __ldg(x + src * vec_per_row + v);
  }
}

}  // namespace

extern "C" {

blade_status_t blade_gilbert_order(int32_t t, int32_t h, int32_t w, int32_t n_text,
                                   int32_t* perm, int64_t perm_len) {
  if (!perm || t < 1 || h < 1 || w < 1 || n_text < 0) return BLADE_ERR_INVALID_ARG;
  const int64_t frame = int64_t(h) * w;
  if (perm_len != int64_t(n_text) + t * frame || perm_len > INT32_MAX) return BLADE_ERR_INVALID_ARG;
  std::vector<int32_t> cells;
  cells.reserve(size_t(frame));
  CurveWriter cw{w, &cells};
  if (w >= h)
    cw.walk(0, 0, w, 0, 0, h);
  else
    cw.walk(0, 0, 0, h, w, 0);
  if (int64_t(cells.size()) != frame) return BLADE_ERR_INVALID_ARG;
  int64_t o = 0;
  for (int32_t s = 0; s < n_text; ++s) perm[o++] = s;
  for (int32_t f = 0; f < t; ++f)
    for (int64_t c = 0; c < frame; ++c) perm[o++] = int32_t(n_text + f * frame + cells[size_t(c)]);
  return BLADE_OK;
}

blade_status_t blade_permute_tokens(const void* x, int64_t BH, int32_t N, int32_t d,
                                    const int32_t* perm, int32_t inverse, void* out,
                                    void* stream) {
  if (!x || !perm || !out || x == out) return BLADE_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(x) & 15u) || (reinterpret_cast<uintptr_t>(out) & 15u))
    return BLADE_ERR_INVALID_ARG;
  if (BH < 1 || N < 1 || d < 8 || d % 8) return BLADE_ERR_INVALID_ARG;
  const int vpr = d / 8;  // 16-byte vectors per token row
  const int64_t total = BH * N * int64_t(vpr);
  const int64_t blocks = (total + 255) / 256;
  const unsigned grid = unsigned(blocks < 148 * 16 ? blocks : 148 * 16);
  permute_tokens_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(x), BH, N, vpr, perm, inverse ? 1 : 0, static_cast<uint4*>(out));
  return cudaGetLastError() == cudaSuccess ? BLADE_OK : BLADE_ERR_CUDA;
}

}  // extern "C"
