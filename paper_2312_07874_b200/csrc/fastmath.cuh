// Branch-free natural logarithm and exponential for the pointwise phases of the entropy projection
// (K1: W(u) and U(w), PAPER App. B).  CUDA's log() / exp() carry a special-case
// branch each, which keeps ptxas from interleaving the evaluations of several nodes of one thread;
// these versions are straight-line code (arguments: positive normal doubles for the logarithm,
// |y| < 700 for the exponential -- admissible states, checked by the caller's `bad` flag), so two
// nodes per thread run as independent instruction streams.
// Accuracy (tests/test_host_fastmath.py, against libm over 2^-60 .. 2^60 and -600 .. 600): <= 2 ulp.
// The header compiles for the host too (the test builds it with g++); it holds no table and no
// constant shared with the oracle.
#pragma once
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define ES_FM_FN __host__ __device__ __forceinline__
#else
#include <math.h>
#define ES_FM_FN static inline
#endif

// Polynomial coefficients: on the device they are read as constant-bank operands of the DFMAs (a
// 64-bit literal costs two UMOV issue slots per use, ~50 per node in the ncu source view)
#define ES_FM_COEFFS                                                                                       \
  {2.0 / 21.0, 2.0 / 19.0, 2.0 / 17.0, 2.0 / 15.0, 2.0 / 13.0, 2.0 / 11.0, 2.0 / 9.0, 2.0 / 7.0, 2.0 / 5.0, \
   2.0 / 3.0, 6.93147180369123816490e-01, 1.90821492927058770002e-10, 1.0 / 87178291200.0,                 \
   1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0, \
   1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 1.44269504088896338700e+00}
#if defined(__CUDACC__)
static __constant__ double es_fm_cdev[25] = ES_FM_COEFFS;
#endif
static const double es_fm_chost[25] = ES_FM_COEFFS;
#if defined(__CUDA_ARCH__)
#define ES_FM_C(i) es_fm_cdev[i]
#else
#define ES_FM_C(i) es_fm_chost[i]
#endif

ES_FM_FN int64_t es_fm_bits(double x) {
#if defined(__CUDA_ARCH__)
  return __double_as_longlong(x);
#else
  int64_t i;
  memcpy(&i, &x, 8);
  return i;
#endif
}
ES_FM_FN double es_fm_double(int64_t i) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(i);
#else
  double x;
  memcpy(&x, &i, 8);
  return x;
#endif
}

// 1 / s for positive normal s: hardware seed and one cubic step (as rcp_nr in rhs2.cuh)
ES_FM_FN double es_fm_rcp(double s) {
#if defined(__CUDA_ARCH__)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  const double e = fma(-s, r, 1.0);
  return fma(r, fma(e, e, e), r);
#else
  return 1.0 / s;
#endif
}

// log(x) = k ln 2 + 2 atanh(f), x = 2^k m, m in [sqrt(1/2), sqrt(2)), f = (m - 1)/(m + 1):
// |f| <= 0.1716, z = f^2 <= 0.02944; atanh series to z^10 (next term z^11/23 < 7e-19)
ES_FM_FN double es_log_pos(double x) {
  const int64_t ix = es_fm_bits(x);
  const int64_t k = (ix - 0x3fe6a09e667f3bcdLL) >> 52;
  const double m = es_fm_double(ix - (int64_t)((uint64_t)k << 52));
  const double kf = (double)(int)k;
  const double a = m - 1.0, b = m + 1.0;  // a exact (Sterbenz)
  const double rb = es_fm_rcp(b);
  double f = a * rb;
  f = fma(fma(-f, b, a), rb, f);  // quotient correction
  const double z = f * f;
  double P = ES_FM_C(0);
#pragma unroll
  for (int q = 1; q < 10; ++q) P = fma(P, z, ES_FM_C(q));
  const double lm = fma(f * z, P, f + f);                    // 2 atanh(f)
  // ln 2 = hi + lo, hi with 32 trailing zero bits: kf * hi exact
  return fma(kf, ES_FM_C(10), fma(kf, ES_FM_C(11), lm));
}

// exp(y) = 2^n exp(r), n = round(y / ln 2), |r| <= 0.3466; Taylor series to r^14 (next term < 1e-19)
ES_FM_FN double es_exp(double y) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: the integer lands in the low mantissa bits
  const double t = fma(y, ES_FM_C(24), magic);
  const double nf = t - magic;
  const int64_t n = (int64_t)(int32_t)(uint32_t)es_fm_bits(t);
  double r = fma(-nf, ES_FM_C(10), y);
  r = fma(-nf, ES_FM_C(11), r);
  double P = ES_FM_C(12);  // 1/14!
#pragma unroll
  for (int q = 13; q < 24; ++q) P = fma(P, r, ES_FM_C(q));  // ... 1/3!
  P = fma(P, r, 0.5);
  const double e = fma(r * r, P, r) + 1.0;  // 1 + r + r^2 P
  return es_fm_double(es_fm_bits(e) + (int64_t)((uint64_t)n << 52));
}
