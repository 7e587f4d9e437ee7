// fexp.cuh -- exp(x) for the generated thread-per-cell mechanism code.
//
// Cody-Waite reduction x = k ln2 + r (|r| <= ln2/2, k = rint(x log2 e) by the
// 1.5 * 2^52 rounding trick), e^r by its degree-12 Taylor polynomial in Horner
// form (truncation r^13/13! <= 1.7e-16 relative: about one ulp), 2^k applied
// by exponent arithmetic.  The coefficients live in __constant__ memory, so
// every DFMA takes them as a constant-bank operand: the library exp spends
// two uniform-register moves per 64-bit coefficient, which doubles the issue
// count of an exp-bound RHS.  x > 708.39 gives +inf, x < -707 gives 0 (no denormal
// results); NaN propagates.  Accuracy is all the RHS parity bar needs
// (|df| <= 1e-12 S, reading R19); the oracle uses its own libm exp.
#pragma once

#ifndef BDFB_FEXP_ESTRIN
#define BDFB_FEXP_ESTRIN 0
#endif

namespace bdfb {

__constant__ double kFexp[15] = {
    0x1.71547652b82fep+0,    // log2(e)
    0x1.62e42fefa39efp-1,    // ln2_hi (ln 2 rounded to double)
    2.319046813846299558e-17,  // ln2_lo = ln 2 - ln2_hi
    1.0 / 479001600.0,       // 1/12!
    1.0 / 39916800.0,        // 1/11!
    1.0 / 3628800.0,         // 1/10!
    1.0 / 362880.0,          // 1/9!
    1.0 / 40320.0,           // 1/8!
    1.0 / 5040.0,            // 1/7!
    1.0 / 720.0,             // 1/6!
    1.0 / 120.0,             // 1/5!
    1.0 / 24.0,              // 1/4!
    1.0 / 6.0,               // 1/3!
    0.5,                     // 1/2!
    1.0};

__device__ __forceinline__ double fexp(double x) {
  const double t = fma(x, kFexp[0], 6755399441055744.0);   // 1.5 * 2^52: low word = rint(x log2 e)
  const double k = t - 6755399441055744.0;
  double r = fma(k, -kFexp[1], x);
  r = fma(k, -kFexp[2], r);
#if BDFB_FEXP_ESTRIN
  // Estrin's scheme: the same degree-12 Taylor polynomial, 5 dependent FMA levels instead of 13 (the RHS is
  // latency-bound on these chains); coefficients c_k = 1/k! (kFexp[15 - k] for k >= 2)
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  const double a0 = fma(r, 1.0, 1.0), a1 = fma(kFexp[12], r, kFexp[13]), a2 = fma(kFexp[10], r, kFexp[11]),
               a3 = fma(kFexp[8], r, kFexp[9]), a4 = fma(kFexp[6], r, kFexp[7]), a5 = fma(kFexp[4], r, kFexp[5]);
  const double b0 = fma(a1, r2, a0), b1 = fma(a3, r2, a2), b2 = fma(a5, r2, a4);
  const double d0 = fma(b1, r4, b0), d1 = fma(kFexp[3], r4, b2);
  const double p = fma(d1, r8, d0);
#else
  double p = fma(kFexp[3], r, kFexp[4]);
#pragma unroll
  for (int i = 5; i < 14; ++i) p = fma(p, r, kFexp[i]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
#endif
  const int ki = __double2loint(t);
  double res = __hiloint2double(__double2hiint(p) + (ki << 20), __double2loint(p));
  // branch-free range handling (a taken branch per exp breaks the instruction
  // prefetch of the straight-line RHS): results beyond the normal range of the
  // scaling saturate to +inf / 0 (x > 708.39: e^x > 2^1022; x < -707: e^x < 2^-1020);
  // NaN propagates through the arithmetic above.
  res = (x > 708.39) ? __longlong_as_double(0x7ff0000000000000ll) : res;
  res = (x < -707.0) ? 0.0 : res;   // keeps k >= -1021: no denormal exponent field
  return res;
}

}  // namespace bdfb
