// Deterministic exp/log/pow for the decode path (device side).
//
// The reference takes exp/log from Eigen packet math and glibc
// (tensor.cpp:346-349, model.cpp:647-648, decode.cpp:18-21, 26-29), whose last
// ulp depends on the build host. These Cephes polynomials use only correctly
// rounded IEEE ops (explicit __fmaf_rn; the library is compiled --fmad=false),
// so the CPU oracle (oracle/detmath.h) reproduces them bit for bit. Accuracy:
// < 1 ulp against libm over the ranges the kernels use.
#pragma once

#include <cstdint>

namespace mtg {

__device__ __forceinline__ float det_expf(float x) {
  if (x != x) return x;
  if (x > 88.72283935546875f) return __int_as_float(0x7f800000);
  if (x < -103.97208404541015625f) return 0.0f;
  const float n = rintf(__fmul_rn(x, 1.44269502162933349609375f));
  float r = __fmaf_rn(n, -0.693359375f, x);
  r = __fmaf_rn(n, 2.12194440e-4f, r);
  const float z = __fmul_rn(r, r);
  float p = 1.9875691500e-4f;
  p = __fmaf_rn(p, r, 1.3981999507e-3f);
  p = __fmaf_rn(p, r, 8.3334519073e-3f);
  p = __fmaf_rn(p, r, 4.1665795894e-2f);
  p = __fmaf_rn(p, r, 1.6666665459e-1f);
  p = __fmaf_rn(p, r, 5.0000001201e-1f);
  p = __fmaf_rn(p, z, r);
  p = __fadd_rn(p, 1.0f);
  const int ni = static_cast<int>(n);
  const int n1 = ni / 2;
  const int n2 = ni - n1;
  p = __fmul_rn(p, __int_as_float((n1 + 127) << 23));
  p = __fmul_rn(p, __int_as_float((n2 + 127) << 23));
  return p;
}

// det_expf for x <= 0 (softmax arguments x - max, -inf allowed): same bits,
// branch-free (both scalings computed, then selected).
__device__ __forceinline__ float det_expf_nonpos(float x) {
  const bool under = x < -103.97208404541015625f;
  x = under ? 0.0f : x;
  const float n = rintf(__fmul_rn(x, 1.44269502162933349609375f));
  float r = __fmaf_rn(n, -0.693359375f, x);
  r = __fmaf_rn(n, 2.12194440e-4f, r);
  const float z = __fmul_rn(r, r);
  float p = 1.9875691500e-4f;
  p = __fmaf_rn(p, r, 1.3981999507e-3f);
  p = __fmaf_rn(p, r, 8.3334519073e-3f);
  p = __fmaf_rn(p, r, 4.1665795894e-2f);
  p = __fmaf_rn(p, r, 1.6666665459e-1f);
  p = __fmaf_rn(p, r, 5.0000001201e-1f);
  p = __fmaf_rn(p, z, r);
  p = __fadd_rn(p, 1.0f);
  const int ni = static_cast<int>(n);
  // Normal result: scaling by 2^n is exact, so adding n to the exponent
  // gives the same bits as the two multiplies.
  const float fast = __int_as_float(__float_as_int(p) + (ni << 23));
  const int n1 = ni / 2;
  const float slow = __fmul_rn(__fmul_rn(p, __int_as_float((n1 + 127) << 23)),
                               __int_as_float((ni - n1 + 127) << 23));
  return under ? 0.0f : (ni >= -125 ? fast : slow);
}

// det_expf_nonpos for x in [-86.5, 0] or NaN: same bits with fewer, full-rate
// instructions. n = rint(x * log2e) via the 1.5 * 2^23 rounding add (round to
// nearest even, like rintf), and 2^n (normal, n >= -125) is built from the
// low bits of that sum, so no FRND / F2I and no subnormal path.
__device__ __forceinline__ float det_expf_nonpos_fast(float x) {
  const float t = __fadd_rn(__fmul_rn(x, 1.44269502162933349609375f), 12582912.0f);
  const float n = __fsub_rn(t, 12582912.0f);
  float r = __fmaf_rn(n, -0.693359375f, x);
  r = __fmaf_rn(n, 2.12194440e-4f, r);
  const float z = __fmul_rn(r, r);
  float p = 1.9875691500e-4f;
  p = __fmaf_rn(p, r, 1.3981999507e-3f);
  p = __fmaf_rn(p, r, 8.3334519073e-3f);
  p = __fmaf_rn(p, r, 4.1665795894e-2f);
  p = __fmaf_rn(p, r, 1.6666665459e-1f);
  p = __fmaf_rn(p, r, 5.0000001201e-1f);
  p = __fmaf_rn(p, z, r);
  p = __fadd_rn(p, 1.0f);
  return __fmul_rn(p, __int_as_float((__float_as_int(t) << 23) + 0x3f800000));
}

// Sequential sum of exp(s[j] - best), j < nv, in column order (P6). `mn` is
// the lane's fminf over its nv values; when every lane of the warp has
// mn - best >= -86.5 the fast exp gives the same bits as det_expf_nonpos.
__device__ __forceinline__ float det_sum_exp(const float* s, int nv, float best, float mn) {
  float sum = 0.0f;
  if (__all_sync(0xffffffffu, __fsub_rn(mn, best) >= -86.5f)) {
#pragma unroll 4
    for (int j = 0; j < nv; ++j) sum = __fadd_rn(sum, det_expf_nonpos_fast(__fsub_rn(s[j], best)));
  } else {
#pragma unroll 4
    for (int j = 0; j < nv; ++j) sum = __fadd_rn(sum, det_expf_nonpos(__fsub_rn(s[j], best)));
  }
  return sum;
}

__device__ __forceinline__ float det_logf(float x) {
  if (x != x) return x;
  if (x < 0.0f) return __int_as_float(0x7fc00000);
  if (x == 0.0f) return __int_as_float(0xff800000);
  if (x == __int_as_float(0x7f800000)) return x;
  uint32_t bits = __float_as_uint(x);
  int eadj = 0;
  if (bits < 0x00800000u) {
    x = __fmul_rn(x, 8388608.0f);
    bits = __float_as_uint(x);
    eadj = -23;
  }
  int e = static_cast<int>((bits >> 23) & 0xffu) - 126 + eadj;
  float m = __uint_as_float((bits & 0x007fffffu) | 0x3f000000u);
  if (m < 0.707106781186547524f) {
    e -= 1;
    m = __fsub_rn(__fadd_rn(m, m), 1.0f);
  } else {
    m = __fsub_rn(m, 1.0f);
  }
  const float z = __fmul_rn(m, m);
  float y = 7.0376836292e-2f;
  y = __fmaf_rn(y, m, -1.1514610310e-1f);
  y = __fmaf_rn(y, m, 1.1676998740e-1f);
  y = __fmaf_rn(y, m, -1.2420140846e-1f);
  y = __fmaf_rn(y, m, 1.4249322787e-1f);
  y = __fmaf_rn(y, m, -1.6668057665e-1f);
  y = __fmaf_rn(y, m, 2.0000714765e-1f);
  y = __fmaf_rn(y, m, -2.4999993993e-1f);
  y = __fmaf_rn(y, m, 3.3333331174e-1f);
  y = __fmul_rn(y, m);
  y = __fmul_rn(y, z);
  const float fe = static_cast<float>(e);
  y = __fmaf_rn(fe, -2.12194440e-4f, y);
  y = __fmaf_rn(z, -0.5f, y);
  float r = __fadd_rn(m, y);
  r = __fmaf_rn(fe, 0.693359375f, r);
  return r;
}

__device__ __forceinline__ float det_powf(float b, float a) {
  if (a == 1.0f) return b;
  if (a == 0.0f) return 1.0f;
  return det_expf(__fmul_rn(a, det_logf(b)));
}

// Lane-strided partials then xor butterfly: every lane ends with the same
// bits (float add is commutative). Order P1 in DESIGN.md §3.
__device__ __forceinline__ float warp_allsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_allmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace mtg
