/*
 * TEST INFRASTRUCTURE (oracle) -- not product code.
 *
 * Deterministic float transcendentals used by the oracle. The reference gets
 * exp/log from Eigen's packet math (pexp) and glibc (std::log, std::pow)
 * (tensor.cpp:346-349, decode.cpp:26-29, decode.cpp:18-21), whose last-ulp
 * behaviour depends on -march. The GPU path fixes them to the Cephes
 * polynomials below, evaluated with explicit fmaf and separately rounded
 * ops only, so host and device produce identical bits. The product's copy
 * lives in paper_2008_04885_b200/csrc/detmath.cuh; tests check the two agree
 * bit for bit and stay within 2 ulp of libm.
 */
#ifndef ORACLE_DETMATH_H_
#define ORACLE_DETMATH_H_

#include <math.h>
#include <stdint.h>
#include <string.h>

static inline float orc_u2f(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint32_t orc_f2u(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}

/* exp(x): Cephes expf range reduction + degree-6 polynomial. */
static inline float orc_expf(float x) {
  if (x != x) return x;
  if (x > 88.72283935546875f) return INFINITY;
  if (x < -103.97208404541015625f) return 0.0f;
  const float n = rintf(x * 1.44269502162933349609375f);
  float r = fmaf(n, -0.693359375f, x);
  r = fmaf(n, 2.12194440e-4f, r);
  const float z = r * r;
  float p = 1.9875691500e-4f;
  p = fmaf(p, r, 1.3981999507e-3f);
  p = fmaf(p, r, 8.3334519073e-3f);
  p = fmaf(p, r, 4.1665795894e-2f);
  p = fmaf(p, r, 1.6666665459e-1f);
  p = fmaf(p, r, 5.0000001201e-1f);
  p = fmaf(p, z, r);
  p = p + 1.0f;
  const int ni = (int)n;
  const int n1 = ni / 2;
  const int n2 = ni - n1;
  p = p * orc_u2f((uint32_t)(n1 + 127) << 23);
  p = p * orc_u2f((uint32_t)(n2 + 127) << 23);
  return p;
}

/* log(x): Cephes logf (mantissa in [sqrt(1/2), sqrt(2)) + degree-8 poly). */
static inline float orc_logf(float x) {
  if (x != x) return x;
  if (x < 0.0f) return NAN;
  if (x == 0.0f) return -INFINITY;
  if (x == INFINITY) return x;
  uint32_t bits = orc_f2u(x);
  int eadj = 0;
  if (bits < 0x00800000u) { /* subnormal */
    x = x * 8388608.0f;
    bits = orc_f2u(x);
    eadj = -23;
  }
  int e = (int)((bits >> 23) & 0xffu) - 126 + eadj;
  float m = orc_u2f((bits & 0x007fffffu) | 0x3f000000u); /* [0.5, 1) */
  if (m < 0.707106781186547524f) {
    e -= 1;
    m = m + m - 1.0f;
  } else {
    m = m - 1.0f;
  }
  const float z = m * m;
  float y = 7.0376836292e-2f;
  y = fmaf(y, m, -1.1514610310e-1f);
  y = fmaf(y, m, 1.1676998740e-1f);
  y = fmaf(y, m, -1.2420140846e-1f);
  y = fmaf(y, m, 1.4249322787e-1f);
  y = fmaf(y, m, -1.6668057665e-1f);
  y = fmaf(y, m, 2.0000714765e-1f);
  y = fmaf(y, m, -2.4999993993e-1f);
  y = fmaf(y, m, 3.3333331174e-1f);
  y = y * m;
  y = y * z;
  const float fe = (float)e;
  y = fmaf(fe, -2.12194440e-4f, y);
  y = fmaf(z, -0.5f, y);
  float r = m + y;
  r = fmaf(fe, 0.693359375f, r);
  return r;
}

/* pow(b, a) for the GNMT penalty (decode.cpp:18-21): exact for a = 1 and
 * a = 0 (as libm), exp(a*log(b)) otherwise. */
static inline float orc_powf(float b, float a) {
  if (a == 1.0f) return b;
  if (a == 0.0f) return 1.0f;
  return orc_expf(a * orc_logf(b));
}

#endif /* ORACLE_DETMATH_H_ */
