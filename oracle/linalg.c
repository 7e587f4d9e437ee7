/*
 * linalg.c -- oracle WRMS norm and dense LU (TEST INFRASTRUCTURE ONLY; see
 * oracle.h).
 */
#include <math.h>
#include "oracle.h"

/*
 * Weighted RMS norm, Eq. 3:  ||v|| = sqrt( (1/N) sum (w_i v_i)^2 ).
 *
 * Reading R15 (summation order is paper-silent): for a cell owned by a group
 * of G lanes, lane l first sums (w_i v_i)^2 over i = l, l+G, l+2G, ... in
 * increasing i; the G partial sums are then combined by an xor butterfly with
 * offsets G/2, ..., 1 (s[l] <- s[l] + s[l ^ off]); the result is s[0].
 * G = 1 is the plain sequential sum.  The order changes only rounding.
 * Pins: tests/test_oracle_primitives.py (S:82-84 examples, homogeneity,
 * brute-force comparison with math.fsum within rounding).
 */
double orc_wrms(int n, const double *v, const double *w, int group)
{
  return sqrt(orc_wrms_sum(n, v, w, group) / (double)n);
}

/* the sum S of Eq. 3 before the division by N and the square root */
double orc_wrms_sum(int n, const double *v, const double *w, int group)
{
  double s[64];
  int G = group < 1 ? 1 : group;
  for (int l = 0; l < G; ++l) {
    double acc = 0.0;
    for (int i = l; i < n; i += G) {
      double p = v[i] * w[i];
      acc = acc + p * p;
    }
    s[l] = acc;
  }
  for (int off = G / 2; off >= 1; off /= 2) {
    double t[64];
    for (int l = 0; l < G; ++l) t[l] = s[l] + s[l ^ off];
    for (int l = 0; l < G; ++l) s[l] = t[l];
  }
  return s[0];
}

/*
 * LU factorisation with partial pivoting ("LU factorization with
 * pivoting"), getrf semantics, listing LU_FACTOR and reading R16:
 *   for k: p = first argmax_{i>=k} |M[i][k]|; piv[k] = p;
 *          M[p][k] == 0 -> singular (returns k+1, recoverable);
 *          swap rows k,p; r = 1/M[k][k]; M[i][k] *= r (i>k);
 *          M[i][j] = fma(-M[i][k], M[k][j], M[i][j])  (i>k, j>k).
 * Pins: brute-force Gaussian elimination (numpy) with identical pivots,
 * SPEC examples S:275-287, backward error <= n*u.
 */
int orc_lu_factor(int n, double *M, int *piv)
{
  for (int k = 0; k < n; ++k) {
    int p = k;
    double amax = fabs(M[k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      double a = fabs(M[i * n + k]);
      if (a > amax) { amax = a; p = i; }
    }
    piv[k] = p;
    if (M[p * n + k] == 0.0) return k + 1;
    if (p != k) {
      for (int j = 0; j < n; ++j) {
        double t = M[k * n + j];
        M[k * n + j] = M[p * n + j];
        M[p * n + j] = t;
      }
    }
    double r = 1.0 / M[k * n + k];
    for (int i = k + 1; i < n; ++i) M[i * n + k] *= r;
    for (int i = k + 1; i < n; ++i)
      for (int j = k + 1; j < n; ++j)
        M[i * n + j] = fma(-M[i * n + k], M[k * n + j], M[i * n + j]);
  }
  return 0;
}

/*
 * Solve with the factors (getrs semantics), listing LU_SOLVE:
 *   swaps b[k] <-> b[piv[k]] in order; unit-L forward substitution in
 *   column (axpy) order with fma; U back substitution in column order with
 *   fma, b[k] multiplied by the correctly rounded reciprocal 1/U[k][k]
 *   (reading R16: one reciprocal per pivot instead of a division per solve).
 */
void orc_lu_solve(int n, const double *LU, const int *piv, double *b)
{
  for (int k = 0; k < n; ++k) {
    int p = piv[k];
    if (p != k) { double t = b[k]; b[k] = b[p]; b[p] = t; }
  }
  for (int k = 0; k < n - 1; ++k)
    for (int i = k + 1; i < n; ++i)
      b[i] = fma(-LU[i * n + k], b[k], b[i]);
  for (int k = n - 1; k > 0; --k) {
    b[k] = b[k] * (1.0 / LU[k * n + k]);
    for (int i = 0; i < k; ++i)
      b[i] = fma(-LU[i * n + k], b[k], b[i]);
  }
  b[0] = b[0] * (1.0 / LU[0]);
}

/* LU_SOLVE exactly as the listing writes it (plain mode): b[k] /= U[k][k]
 * (true division) instead of the multiplication by 1/U[k][k] of reading R16. */
void orc_lu_solve_div(int n, const double *LU, const int *piv, double *b)
{
  for (int k = 0; k < n; ++k) {
    int p = piv[k];
    if (p != k) { double t = b[k]; b[k] = b[p]; b[p] = t; }
  }
  for (int k = 0; k < n - 1; ++k)
    for (int i = k + 1; i < n; ++i)
      b[i] = fma(-LU[i * n + k], b[k], b[i]);
  for (int k = n - 1; k > 0; --k) {
    b[k] = b[k] / LU[k * n + k];
    for (int i = 0; i < k; ++i)
      b[i] = fma(-LU[i * n + k], b[k], b[i]);
  }
  b[0] = b[0] / LU[0];
}

/* Eq. 7: typical value = midpoint of the component's range over the whole domain. */
void orc_typical_values(int n, int64_t ncells, const double *y, double *tv)
{
  for (int k = 0; k < n; ++k) {
    double lo = y[(int64_t)k * ncells], hi = lo;
    for (int64_t c = 1; c < ncells; ++c) {
      const double v = y[(int64_t)k * ncells + c];
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
    tv[k] = 0.5 * (lo + hi);
  }
}

/* Eq. 7: atol_i = eta * tv_i, with the floor of S:99 */
void orc_atol_from_typical(int n, const double *tv, double eta, double floor_, double *atol)
{
  for (int k = 0; k < n; ++k) atol[k] = fmax(eta * tv[k], floor_);
}
