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
  double p = fma(kFexp[3], r, kFexp[4]);
#pragma unroll
  for (int i = 5; i < 14; ++i) p = fma(p, r, kFexp[i]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
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
