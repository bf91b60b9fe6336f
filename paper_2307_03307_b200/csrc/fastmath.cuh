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

#if defined(__CUDA_ARCH__)
#define MWU_IF(k) kMwuInvFact[k]
#else
#define MWU_IF(k) kMwuInvFact[k]
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
