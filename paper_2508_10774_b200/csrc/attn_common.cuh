// attn_common.cuh — pieces shared by the two tcgen05 attention kernels
// (attn_tc.cu: one query block per CTA; attn_tc2.cu: two per CTA).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"

namespace blade {
namespace attn {

// 2^x for a pair on the FMA pipe: x = n + f with n = rint(x) (1.5 * 2^23
// trick), f in [-1/2, 1/2], 2^f by a degree-3 minimax polynomial (|rel err|
// < 7.5e-5, far below the bf16 rounding P gets next), n added to the exponent
// field.  Packed fp32x2 ops: 6 FMA-pipe slots for two exponentials.
BLADE_DEVINL float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = add2(x, make_float2(12582912.f, 12582912.f));
  const float2 n = add2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = fma2(n, make_float2(-1.f, -1.f), x);
  float2 p = fma2(f, make_float2(5.517165314e-2f, 5.517165314e-2f),
                  make_float2(2.426111615e-1f, 2.426111615e-1f));
  p = fma2(p, f, make_float2(6.932609919e-1f, 6.932609919e-1f));
  p = fma2(p, f, make_float2(9.999280713e-1f, 9.999280713e-1f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// fp32(1/sqrt(d)) * fp32(log2 e) as the host computes it for the default
// scale; baking it in lets the exponent FFMA use its immediate form.
template <int D>
struct DefaultScale;
template <>
struct DefaultScale<128> {
  static constexpr float kScaleLog2 = 0.088388346f * 1.44269502f;
};
template <>
struct DefaultScale<64> {
  static constexpr float kScaleLog2 = 0.125f * 1.44269502f;
};

// Global tokens of ASA_GT: N_g pooled K/V rows attended by every
// query after its kept blocks, as ceil(N_g/128) extra tiles with the additive
// bias ln(n_w) (readings R-18..R-20), applied in raw-score units (/ scale).
struct GtArgs {
  int Ng;             // number of global tokens (0: plain ASA)
  float bias_full;    // ln(n) / scale      (full windows)
  float bias_last;    // ln(n_last) / scale (the last, possibly partial, window)
};

}  // namespace attn
}  // namespace blade
