// Deterministic transcendental functions built only from correctly rounded
// IEEE operations (+ - * / fmaf fma rint and exact exponent scaling), so the
// same source gives bit-identical results on the host (gcc, -ffp-contract=off)
// and on the device (nvcc -fmad=false). The fitness stage needs this: greedy
// CTC tokens, edit distances and LER must be bit-exact against the CPU
// restatement in oracle/, which re-derives the same algorithm independently.
//
// Algorithm (documented in DESIGN.md, "fitness numerics"):
//   expf : clamp to [-87, 88]; n = rint(x*log2e); r = x - n*ln2 (Cody-Waite,
//          two fmaf); p = degree-7 Taylor polynomial in r (fmaf Horner);
//          result = p * 2^n (exact exponent scaling).
//   sigm : 1 / (1 + expf(-x))
//   tanh : s = sign(x); e = expf(-2|x|); s * (1 - e) / (1 + e)
//   log1p_d (fp64, feature normalisation): y = 1 + v; y = m * 2^e with m in
//          [sqrt(1/2), sqrt(2)); f = m - 1; s = f / (2 + f);
//          log(m) = 2s * sum_{k=0..11} s^(2k)/(2k+1) (fma Horner); + e*ln2.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define TOBF_HD __host__ __device__ __forceinline__
#else
#define TOBF_HD static inline
#endif

TOBF_HD float tobf_bits2f(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

TOBF_HD double tobf_bits2d(uint64_t u) {
  double f;
  memcpy(&f, &u, 8);
  return f;
}

TOBF_HD uint64_t tobf_d2bits(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
}

TOBF_HD float tobf_expf(float x) {
  if (x > 88.0f) x = 88.0f;
  if (x < -87.0f) x = -87.0f;
  const float t = x * 1.44269504088896341f;
  const float n = rintf(t);
  float r = fmaf(n, -0.693145751953125f, x);
  r = fmaf(n, -1.428606765330187045e-06f, r);
  float p = 1.98412698412698413e-04f;  // 1/5040
  p = fmaf(p, r, 1.38888888888888889e-03f);  // 1/720
  p = fmaf(p, r, 8.33333333333333333e-03f);  // 1/120
  p = fmaf(p, r, 4.16666666666666667e-02f);  // 1/24
  p = fmaf(p, r, 1.66666666666666667e-01f);  // 1/6
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  const int ni = (int)n;  // in [-126, 127] after the clamp
  const float scale = tobf_bits2f((uint32_t)(ni + 127) << 23);
  return p * scale;
}

TOBF_HD float tobf_sigmoid(float x) { return 1.0f / (1.0f + tobf_expf(-x)); }

TOBF_HD float tobf_tanh(float x) {
  const float ax = fabsf(x);
  const float e = tobf_expf(-2.0f * ax);
  const float t = (1.0f - e) / (1.0f + e);
  return x < 0.0f ? -t : t;
}

// log(1 + v) for v >= 0 in fp64 (feature normalisation), IEEE ops only.
TOBF_HD double tobf_log1p_d(double v) {
  const double y = 1.0 + v;
  uint64_t bits = tobf_d2bits(y);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  double m = tobf_bits2d((bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL);  // [1, 2)
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e += 1;
  }
  const double f = m - 1.0;
  const double s = f / (2.0 + f);
  const double s2 = s * s;
  double p = 1.0 / 23.0;
  p = fma(p, s2, 1.0 / 21.0);
  p = fma(p, s2, 1.0 / 19.0);
  p = fma(p, s2, 1.0 / 17.0);
  p = fma(p, s2, 1.0 / 15.0);
  p = fma(p, s2, 1.0 / 13.0);
  p = fma(p, s2, 1.0 / 11.0);
  p = fma(p, s2, 1.0 / 9.0);
  p = fma(p, s2, 1.0 / 7.0);
  p = fma(p, s2, 1.0 / 5.0);
  p = fma(p, s2, 1.0 / 3.0);
  p = fma(p, s2, 1.0);
  const double lm = 2.0 * s * p;
  return fma((double)e, 0.6931471805599453, lm);
}
