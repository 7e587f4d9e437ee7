/*
 * krylov.c -- oracle scaled GMRES for the inexact Newton-Krylov approaches
 * 1A/1B (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * Paper: Table 1 rows 1A/1B ("Inexact Newton | GMRES | Numerical
 * Jv-product"); the scaled system of Eq. 5, A~ = S1 P1^-1 A P2^-1
 * S2^-1, b~ = S1 P1^-1 b, x~ = S2 P2 x, with S1 = S2 = diag(w_i) (the Eq. 3
 * weights) and no preconditioner (P1 = P2 = I: "development of an
 * effective ... preconditioner ... remains an area of ongoing research",
 * P:396); the stopping test of Eq. 6, ||b~ - A~ x~||_2 <
 * c_l (c_eps eps), with the residual norm "from the rotations used to solve
 * the least-squares problem" (Saad 2003).
 *
 * Algorithm: GMRES with modified Gram-Schmidt Arnoldi and Givens rotations
 * (Saad 2003, Alg. 6.9), no restarts, zero initial guess, in the order of
 * SUNDIALS' SPGMR (the implementation the paper runs, reading R29 in
 * DESIGN.md): V0 = S1 b / beta; per iteration l: V_{l+1} = S1 A S2^-1 V_l,
 * MGS against V_0..V_l (with the SUNModifiedGS re-orthogonalisation test,
 * FACTOR = 1000), Givens update of column l of the Hessenberg matrix,
 * rho = |prod_k s_k| beta; converged when rho <= delta; the correction
 * x = S2^-1 sum_k y_k V_k from the rotated least-squares system.  If the cap
 * maxl is reached with rho < beta the best iterate is returned (RES_REDUCED).
 *
 * Pins (tests/test_oracle_krylov.py): A = I converges in one iteration with
 * x = b; a diagonal A with k distinct eigenvalues converges in <= k
 * iterations; the rotation residual equals the explicitly formed
 * ||S1 (b - A x_k)||_2 at every k; x_k is the
 * least-squares minimiser over the Krylov space built independently with
 * numpy; scaled vs unscaled back-transform consistency.
 */
#include <math.h>
#include "oracle.h"

#define GS_FACTOR 1000.0

static double dot(int n, const double *x, const double *y)
{
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = s + x[i] * y[i];
  return s;
}

/* modified Gram-Schmidt of V[k] against V[i0..k-1] (SUNModifiedGS); H column k-1 */
static void mgs(int n, double V[][ORC_NMAX], double H[][ORC_MAXL], int k, int p, double *new_vk_norm)
{
  const int km1 = k - 1, i0 = k - p > 0 ? k - p : 0;
  const double vk_norm = sqrt(dot(n, V[k], V[k]));
  for (int i = i0; i < k; ++i) {
    H[i][km1] = dot(n, V[i], V[k]);
    for (int j = 0; j < n; ++j) V[k][j] = V[k][j] + (-H[i][km1]) * V[i][j];
  }
  *new_vk_norm = sqrt(dot(n, V[k], V[k]));
  /* re-orthogonalise only if the new vector is tiny relative to the input */
  double temp = GS_FACTOR * vk_norm;
  if ((temp + (*new_vk_norm)) != temp) return;
  double new_norm_2 = 0.0;
  for (int i = i0; i < k; ++i) {
    const double new_product = dot(n, V[i], V[k]);
    temp = GS_FACTOR * H[i][km1];
    if ((temp + new_product) == temp) continue;
    H[i][km1] = H[i][km1] + new_product;
    for (int j = 0; j < n; ++j) V[k][j] = V[k][j] + (-new_product) * V[i][j];
    new_norm_2 = new_norm_2 + new_product * new_product;
  }
  if (new_norm_2 != 0.0) {
    const double np = (*new_vk_norm) * (*new_vk_norm) - new_norm_2;
    *new_vk_norm = (np > 0.0) ? sqrt(np) : 0.0;
  }
}

/* Givens update of Hessenberg column l (SUNQRfact, incremental): the previous
 * rotations, then a new one zeroing H[l+1][l].  Returns 1 if the new diagonal is 0. */
static int qrfact(double H[][ORC_MAXL], double *giv, int l)
{
  for (int k = 0; k < l; ++k) {
    const double c = giv[2 * k], s = giv[2 * k + 1];
    const double t1 = H[k][l], t2 = H[k + 1][l];
    H[k][l] = c * t1 - s * t2;
    H[k + 1][l] = s * t1 + c * t2;
  }
  const double t1 = H[l][l], t2 = H[l + 1][l];
  double c, s;
  if (t2 == 0.0) {
    c = 1.0;
    s = 0.0;
  } else if (fabs(t2) >= fabs(t1)) {
    const double t3 = t1 / t2;
    s = -1.0 / sqrt(1.0 + t3 * t3);
    c = -s * t3;
  } else {
    const double t3 = t2 / t1;
    c = 1.0 / sqrt(1.0 + t3 * t3);
    s = -c * t3;
  }
  giv[2 * l] = c;
  giv[2 * l + 1] = s;
  H[l][l] = c * t1 - s * t2;
  return H[l][l] == 0.0;
}

/* Q g, then back substitution R y = Q g (SUNQRsol); g[0..k] in, y = g[0..k-1] out */
static int qrsol(int k, double H[][ORC_MAXL], const double *giv, double *g)
{
  for (int j = 0; j < k; ++j) {
    const double c = giv[2 * j], s = giv[2 * j + 1];
    const double t1 = g[j], t2 = g[j + 1];
    g[j] = c * t1 - s * t2;
    g[j + 1] = s * t1 + c * t2;
  }
  for (int j = k - 1; j >= 0; --j) {
    if (H[j][j] == 0.0) return 1;
    g[j] = g[j] / H[j][j];
    for (int i = 0; i < j; ++i) g[i] = g[i] - g[j] * H[i][j];
  }
  return 0;
}

int orc_gmres(int n, int maxl, orc_atimes_fn atimes, void *ctx, const double *b, const double *s1,
              const double *s2, double delta, double *x, int *nli, double *res_norm)
{
  double V[ORC_MAXL + 1][ORC_NMAX], H[ORC_MAXL + 1][ORC_MAXL], giv[2 * ORC_MAXL], g[ORC_MAXL + 1];
  double vt[ORC_NMAX], xc[ORC_NMAX];
  if (maxl < 1) maxl = 1;
  if (maxl > ORC_MAXL) maxl = ORC_MAXL;
  *nli = 0;
  for (int i = 0; i < n; ++i) x[i] = 0.0;
  /* r0 = b (x0 = 0), V0 = S1 r0, beta = ||V0||_2 */
  for (int i = 0; i < n; ++i) V[0][i] = s1 ? s1[i] * b[i] : b[i];
  const double beta = sqrt(dot(n, V[0], V[0]));
  *res_norm = beta;
  if (beta <= delta) return ORC_GMRES_SUCCESS;
  for (int i = 0; i <= maxl; ++i)
    for (int j = 0; j < maxl; ++j) H[i][j] = 0.0;
  double rot = 1.0, rho = beta;
  for (int i = 0; i < n; ++i) V[0][i] = (1.0 / beta) * V[0][i];
  int converged = 0, kdim = 0;
  for (int l = 0; l < maxl; ++l) {
    (*nli)++;
    kdim = l + 1;
    /* V_{l+1} = S1 A S2^-1 V_l */
    for (int i = 0; i < n; ++i) vt[i] = s2 ? V[l][i] / s2[i] : V[l][i];
    const int r = atimes(ctx, vt, V[l + 1]);
    if (r != 0) return r < 0 ? ORC_GMRES_ATIMES_FAIL_UNREC : ORC_GMRES_ATIMES_FAIL_REC;
    if (s1)
      for (int i = 0; i < n; ++i) V[l + 1][i] = s1[i] * V[l + 1][i];
    mgs(n, V, H, l + 1, maxl, &H[l + 1][l]);
    if (qrfact(H, giv, l)) return ORC_GMRES_QRFACT_FAIL;
    rot = rot * giv[2 * l + 1];
    rho = fabs(rot * beta);
    *res_norm = rho;
    if (rho <= delta) {
      converged = 1;
      break;
    }
    for (int i = 0; i < n; ++i) V[l + 1][i] = (1.0 / H[l + 1][l]) * V[l + 1][i];
  }
  g[0] = beta;
  for (int i = 1; i <= kdim; ++i) g[i] = 0.0;
  if (qrsol(kdim, H, giv, g)) return ORC_GMRES_QRSOL_FAIL;
  for (int i = 0; i < n; ++i) xc[i] = 0.0;
  for (int k = 0; k < kdim; ++k)
    for (int i = 0; i < n; ++i) xc[i] = xc[i] + g[k] * V[k][i];
  if (converged || rho < beta) {
    for (int i = 0; i < n; ++i) x[i] = s2 ? xc[i] / s2[i] : xc[i];
    return converged ? ORC_GMRES_SUCCESS : ORC_GMRES_RES_REDUCED;
  }
  return ORC_GMRES_CONV_FAIL;
}
