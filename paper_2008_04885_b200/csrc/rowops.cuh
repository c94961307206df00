// Row-level float helpers shared by the LayerNorm / quantize kernels and the
// small-batch GEMV kernels, so every producer of an operand rounds the same
// way: int8 quantization (quant.cpp:108-122) and the LayerNorm arithmetic
// (tensor.cpp:368-387) with P1 warp sums.
#pragma once

#include <cstdint>

#include "detmath.cuh"

namespace mtg {

// quant.cpp:113-118
__device__ __forceinline__ int8_t quant1(float x, float scale) {
  float v = roundf(__fmul_rn(x, scale));
  v = fminf(127.0f, fmaxf(-127.0f, v));
  return static_cast<int8_t>(v);
}
// quant1 for values whose row max gave the scale (|x * scale| <= 127 up to
// two roundings, so the clamp never binds): roundf as nvcc lowers it --
// x + copysign(0.5, x) rounded toward zero, truncated -- without the clamp
// and the FRND (F2I truncates). Same result for every finite x; a row with a
// non-finite value is an error either way (quant.cpp:110-112).
__device__ __forceinline__ int quant1_in_range(float x, float scale) {
  const float p = __fmul_rn(x, scale);
  return __float2int_rz(__fadd_rz(p, copysignf(0.5f, p)));
}
__device__ __forceinline__ float qscale_of(float max_abs) {
  return max_abs == 0.0f ? 1.0f : __fdiv_rn(127.0f, max_abs);
}

// LayerNorm of one row held by a warp in registers (value c = lane + 32 i,
// n <= 32*KPL): mean and population variance by P1 sums, eps 1e-5, then
// ((x - mu) * inv) * g + b. Returns the row's max |y| (all lanes) and sets
// *bad when any output is non-finite (lane-local).
template <int KPL>
__device__ __forceinline__ float ln_normalize_regs(float (&xv)[KPL], const float (&gv)[KPL],
                                                   const float (&bv)[KPL], int n, int lane,
                                                   int* bad) {
  float part = 0.0f;
#pragma unroll
  for (int i = 0; i < KPL; ++i)
    if (lane + 32 * i < n) part = __fadd_rn(part, xv[i]);
  const float nf = static_cast<float>(n);
  const float mu = __fdiv_rn(warp_allsum(part), nf);
  float part2 = 0.0f;
#pragma unroll
  for (int i = 0; i < KPL; ++i)
    if (lane + 32 * i < n) {
      const float dv = __fsub_rn(xv[i], mu);
      part2 = __fadd_rn(part2, __fmul_rn(dv, dv));
    }
  const float var = __fdiv_rn(warp_allsum(part2), nf);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  float mx = 0.0f;
  int b = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int c = lane + 32 * i;
    if (c < n) {
      xv[i] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xv[i], mu), inv), gv[i]), bv[i]);
      mx = fmaxf(mx, fabsf(xv[i]));
      b |= !isfinite(xv[i]);
    }
  }
  *bad = b;
  return warp_allmax(mx);
}

}  // namespace mtg
