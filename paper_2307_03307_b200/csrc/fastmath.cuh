// fastmath.cuh — fp64 exp / expm1 for the hot loops, from ONE argument reduction and ONE
// polynomial, without the special-case branches of the libdevice versions.
//
//   x = k ln2 + r,  |r| <= ln2/2 (Cody-Waite split ln2 = hi + lo, hi with 32 significant bits)
//   p = expm1(r)    (Taylor series to r^14: truncation < 2e-17 relative on |r| <= 0.3466)
//   exp(x)   = 2^k (1 + p)            = fma(2^k, p, 2^k)
//   expm1(x) = 2^k p + (2^k - 1)      = fma(2^k, p, 2^k - 1)   (k = 0: exactly p)
// Both results are accurate to a few ulps relative to themselves for every finite x, so a
// caller needing both (the covering side of the step search: e^{-eta a d} and its expm1) gets
// them from one evaluation instead of choosing between two libm calls per row.
// Compiled by nvcc for the kernels and by g++ for the CPU accuracy test
// (tests/test_fastmath.py checks them against mpmath to 4 ulps).
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define MWU_HD __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define MWU_FMA(a, b, c) __fma_rn(a, b, c)
#else
#define MWU_FMA(a, b, c) fma(a, b, c)
#endif
#else
#define MWU_HD inline
#define MWU_FMA(a, b, c) fma(a, b, c)
#endif

namespace mwu {

MWU_HD double mwu_pow2i(int k) {  // 2^k for -1022 <= k <= 1023
  const uint64_t b = (uint64_t)(k + 1023) << 52;
  double r;
#if defined(__CUDA_ARCH__)
  r = __longlong_as_double((long long)b);
#else
  memcpy(&r, &b, 8);
#endif
  return r;
}

// Taylor coefficients 1/k!, k = 2..14 (device: constant bank, so the polynomial's FMAs read
// them as c[] operands instead of materialising 64-bit immediates every row)
#if defined(__CUDACC__)
__constant__ double kMwuInvFact[13] = {
#else
static const double kMwuInvFact[13] = {
#endif
    0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0, 1.0 / 720.0, 1.0 / 5040.0, 1.0 / 40320.0, 1.0 / 362880.0,
    1.0 / 3628800.0, 1.0 / 39916800.0, 1.0 / 479001600.0, 1.0 / 6227020800.0, 1.0 / 87178291200.0};

#if defined(__CUDACC__) && !defined(__CUDA_ARCH__)
// host pass of nvcc: the __constant__ array is device memory; read a host copy
static const double kMwuInvFactH[13] = {
    0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0, 1.0 / 720.0, 1.0 / 5040.0, 1.0 / 40320.0, 1.0 / 362880.0,
    1.0 / 3628800.0, 1.0 / 39916800.0, 1.0 / 479001600.0, 1.0 / 6227020800.0, 1.0 / 87178291200.0};
#define MWU_IF(k) kMwuInvFactH[k]
#else
#define MWU_IF(k) kMwuInvFact[k]
#endif

// constants of the table-driven exp (device: constant bank operands instead of a pair of
// uniform-register moves per 64-bit immediate and use)
#if defined(__CUDACC__)
__constant__ double kMwuTabC[8] = {
#else
static const double kMwuTabC[8] = {
#endif
    709.78, 369.3299304675746, 0.00270760617331689, 7.453964567463233e-13,
    1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 8.673617379884035e-19};
#if defined(__CUDA_ARCH__)
#define MWU_TC(k) kMwuTabC[k]
#else
#define MWU_TC(k) (k == 0 ? 709.78 : k == 1 ? 369.3299304675746 : k == 2 ? 0.00270760617331689 \
                   : k == 3 ? 7.453964567463233e-13 : k == 4 ? 1.0 / 120.0 : k == 5 ? 1.0 / 24.0 \
                   : k == 6 ? 1.0 / 6.0 : 8.673617379884035e-19)
#endif

// p = expm1(r) for |r| <= ~0.35
MWU_HD double mwu_expm1_reduced(double r) {
  double t = MWU_IF(12);                         // 1/14!
  t = MWU_FMA(t, r, MWU_IF(11));                 // 1/13!
  t = MWU_FMA(t, r, MWU_IF(10));
  t = MWU_FMA(t, r, MWU_IF(9));
  t = MWU_FMA(t, r, MWU_IF(8));
  t = MWU_FMA(t, r, MWU_IF(7));
  t = MWU_FMA(t, r, MWU_IF(6));
  t = MWU_FMA(t, r, MWU_IF(5));
  t = MWU_FMA(t, r, MWU_IF(4));
  t = MWU_FMA(t, r, MWU_IF(3));
  t = MWU_FMA(t, r, MWU_IF(2));
  t = MWU_FMA(t, r, MWU_IF(1));
  t = MWU_FMA(t, r, MWU_IF(0));
  const double r2 = r * r;
  return MWU_FMA(t, r2, r);                      // r + r^2 (1/2 + r/6 + ...)
}

// (expm1(x), exp(x)) for finite x (and x = -inf).
MWU_HD void mwu_expm1_exp(double x, double& em, double& q) {
  if (!(x >= -745.5)) { em = -1.0; q = 0.0; return; }
  if (x > 709.78) { em = INFINITY; q = INFINITY; return; }
  const double kd = rint(x * 1.4426950408889634);
  double r = MWU_FMA(-kd, 6.93147180369123816490e-01, x);   // ln2_hi (exact product)
  r = MWU_FMA(-kd, 1.90821492927058770002e-10, r);          // ln2_lo
  const double p = mwu_expm1_reduced(r);
  const int k = (int)kd;
  if (k >= -1021) {
    const double s = mwu_pow2i(k);
    q = MWU_FMA(s, p, s);
    em = (k == 0) ? p : MWU_FMA(s, p, s - 1.0);
  } else {                                                   // subnormal exp: two-step scaling
    const double s = mwu_pow2i(k + 60);
    q = MWU_FMA(s, p, s) * 8.673617379884035e-19;            // * 2^-60
    em = -1.0;
  }
}

// exp(x) from a 256-entry table T[j] = 2^(j/256) (host-filled by mwu_exp_table, kept by the
// caller in shared memory) and a degree-5 polynomial on |r| <= ln2/512: half the dependent FMA
// chain of mwu_expm1_exp (the column kernel is bound by that latency).
MWU_HD void mwu_exp_table(double* T) {
  for (int j = 0; j < 256; ++j) T[j] = exp2((double)j / 256.0);
}
// host: T[i] = 2^((i-128)/256) and T[i] - 1 as an unevaluated hi + lo pair (long double)
inline void mwu_expm1_tables(double* T, double* Mh, double* Ml) {
  for (int i = 0; i < 256; ++i) {
    const int j = i - 128;
    const long double t = exp2l((long double)j / 256.0L);
    T[i] = (double)t;
    const long double m = t - 1.0L;
    Mh[i] = (double)m;
    Ml[i] = (double)(m - (long double)Mh[i]);
  }
}

// (expm1(x), exp(x)) from the 256-entry tables (T, T - 1 as hi + lo; j in [-128, 128), so
// |x| < ln2/2 needs no 2^k scaling and expm1 suffers no cancellation) and a degree-5
// polynomial: both accurate relative to themselves, with half the dependent FMA chain of
// mwu_expm1_exp.
MWU_HD void mwu_expm1_exp_tab(double x, const double* T, const double* Mh, const double* Ml, double& em, double& q) {
  if (!(x >= -745.5)) { em = -1.0; q = 0.0; return; }
  if (x > 709.78) { em = INFINITY; q = INFINITY; return; }
  const double kd = rint(x * 369.3299304675746);              // 256 / ln2
  double r = MWU_FMA(-kd, 0.00270760617331689, x);             // ln2/256 hi, 32 bits (exact product)
  r = MWU_FMA(-kd, 7.453964567463233e-13, r);                  // ln2/256 lo
  const int ki = (int)kd;
  const int i = ((ki + 128) & 255), k = (ki - (i - 128)) / 256;   // kd = 256 k + (i - 128)
  double p = 1.0 / 120.0;
  p = MWU_FMA(p, r, 1.0 / 24.0);
  p = MWU_FMA(p, r, 1.0 / 6.0);
  p = MWU_FMA(p, r, 0.5);
  p = MWU_FMA(p, r * r, r);                                    // expm1(r)
  const double t = T[i];
  const double tp = t * p;
  const double e0 = Mh[i] + (tp + Ml[i]);                      // 2^(j/256) e^r - 1
  if (k >= -1021) {
    const double s = mwu_pow2i(k);
    q = MWU_FMA(t, p, t) * s;
    em = (k == 0) ? e0 : MWU_FMA(s, e0, s - 1.0);
  } else {
    q = (MWU_FMA(t, p, t) * mwu_pow2i(k + 60)) * 8.673617379884035e-19;
    em = -1.0;
  }
}
MWU_HD double mwu_exp_tab(double x, const double* T) {
  if (!(x >= -745.5)) return 0.0;
  if (x > MWU_TC(0)) return INFINITY;
  const double kd = rint(x * MWU_TC(1));                       // 256 / ln2
  double r = MWU_FMA(-kd, MWU_TC(2), x);                       // ln2/256 hi, 32 bits (exact product)
  r = MWU_FMA(-kd, MWU_TC(3), r);                              // ln2/256 lo
  const int ki = (int)kd;
  const int j = ki & 255, k = (ki - j) / 256;                  // kd = 256 k + j, 0 <= j < 256
  double p = MWU_TC(4);
  p = MWU_FMA(p, r, MWU_TC(5));
  p = MWU_FMA(p, r, MWU_TC(6));
  p = MWU_FMA(p, r, 0.5);
  p = MWU_FMA(p, r * r, r);                                    // expm1(r)
  const double t = T[j];
  const double m = MWU_FMA(t, p, t);                           // 2^(j/256) e^r
  if (k >= -1021) return m * mwu_pow2i(k);
  return (m * mwu_pow2i(k + 60)) * MWU_TC(7);
}

MWU_HD double mwu_exp(double x) {
  double em, q;
  mwu_expm1_exp(x, em, q);
  return q;
}

MWU_HD double mwu_expm1(double x) {
  double em, q;
  mwu_expm1_exp(x, em, q);
  return em;
}

}  // namespace mwu
