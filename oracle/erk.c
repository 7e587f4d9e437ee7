/*
 * erk.c -- oracle explicit adaptive Runge-Kutta integrator for ONE cell
 * (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * Paper: "explicit methods ... provide similar adaptivity in internal time
 * step size, but employ fixed order schemes ... they do not require algebraic
 * solvers"; the experiment uses "a fourth-order explicit method" from
 * ARKODE whose per-step cost is "5.2 RHS evaluations per step"
 * (five stages plus retries).  SURVEY row f4.  The paper names no tableau;
 * reading R30 takes ARKODE's default fourth-order ERK, the
 * Zonneveld 5-stage 4(3) pair:
 *
 *   c = (0, 1/2, 1/2, 1, 3/4)
 *   a21 = 1/2;  a32 = 1/2;  a43 = 1;  a5j = (5/32, 7/32, 13/32, -1/32)
 *   b  = (1/6, 1/3, 1/3, 1/6, 0)                 (order 4: classical RK4)
 *   b^ = (-1/2, 7/3, 7/3, 13/6, -16/3)           (order 3 embedding)
 *   e = b - b^ = (2/3, -2, -2, -2, 16/3)
 *
 * Step from (t, y) with h (all models are autonomous, so the c_i only enter
 * through t):  k_i = f(t + c_i h, y + h sum_{j<i, a_ij != 0} a_ij k_j) (the
 * sum in increasing j, starting from the first nonzero term);
 * y_new = y + h sum_{b_j != 0} b_j k_j;  err = h sum_j e_j k_j.
 *
 * Control (reading R30): weights w = 1/(rtol|y_n| + atol) of Eq. 3 at the
 * step's start; dsm = ||err||_WRMS; accept iff dsm <= 1;
 * eta = SAFETY / dsm^(1/4) (the estimate is O(h^4): exponent 1/(p^+1), p^ = 3),
 * capped at ETAMX1 = 1e4 on the first step, ETAMX = 10 afterwards and 1 right
 * after a failure; on rejection eta = max(ETAMIN, SAFETY / dsm^(1/4)),
 * MXNEF = 7 failures in one step end the cell with ERR_FAILURE; a recoverable
 * RHS failure in a stage cuts h by ETACF = 1/4 (MXNCF = 10 in one step:
 * RHS_FAIL).  k1 = f(t_n, y_n) is reused across the retries of a step.
 * Initial step (o->h0 == 0): Hairer-Wanner (Solving ODEs I, II.4) with WRMS
 * norms: d0 = ||y0||, d1 = ||f0||, h0 = 0.01 d0/d1 (1e-6 if either < 1e-5),
 * d2 = ||f(t0 + h0, y0 + h0 f0) - f0|| / h0, h1 = (0.01/max(d1, d2))^(1/5)
 * (max(1e-6, 1e-3 h0) if max(d1, d2) <= 1e-15), h = min(100 h0, h1), clipped
 * to tf - t0 and hmax.  Roots x^(1/4) = sqrt(sqrt(x)) and x^(1/5) by the
 * R25 root (orc_root), so that CPU and GPU take identical decisions.
 *
 * Pins (tests/test_oracle_erk.py): one step on y' = lambda y equals the
 * degree-4 Taylor polynomial of e^{h lambda} (RK4's stability function)
 * exactly up to rounding; global order 4 +- 0.25 at fixed h (SPEC AC2,
 * S:596); the error estimate is O(h^4) (ratio 16 on halving h); adaptive runs
 * on y' = lambda y meet the tolerance against the closed form; the
 * explicit-vs-implicit direction of P:426 (SPEC AC4) on an ignition
 * cell.
 */
#include <float.h>
#include <math.h>
#include <string.h>
#include "oracle.h"

#define ERK_SAFETY 0.9
#define ERK_ETAMX1 1e4
#define ERK_ETAMX 10.0
#define ERK_ETAMIN 0.1
#define ERK_ETACF 0.25
#define ERK_MXNEF 7
#define ERK_MXNCF 10
#define ERK_UROUND DBL_EPSILON

static const double A21 = 0.5, A32 = 0.5, A43 = 1.0;
static const double A51 = 5.0 / 32.0, A52 = 7.0 / 32.0, A53 = 13.0 / 32.0, A54 = -1.0 / 32.0;
static const double C2 = 0.5, C3 = 0.5, C4 = 1.0, C5 = 0.75;

int orc_erk_step(const orc_problem *p, double t, double h, const double *y, const double *k1in, double *ynew,
                 double *err, int *nfe)
{
  const int n = p->n;
  const double B1 = 1.0 / 6.0, B2 = 1.0 / 3.0, B3 = 1.0 / 3.0, B4 = 1.0 / 6.0;
  const double E1 = 2.0 / 3.0, E2 = -2.0, E3 = -2.0, E4 = -2.0, E5 = 16.0 / 3.0;
  double k[5][ORC_NMAX], ys[ORC_NMAX];
  int r;
  *nfe = 0;
  if (k1in) {
    memcpy(k[0], k1in, sizeof(double) * n);
  } else {
    r = orc_rhs(p, t, y, k[0]);
    (*nfe)++;
    if (r) return r;
  }
  for (int i = 0; i < n; ++i) ys[i] = h * (A21 * k[0][i]) + y[i];
  r = orc_rhs(p, t + C2 * h, ys, k[1]);
  (*nfe)++;
  if (r) return r;
  for (int i = 0; i < n; ++i) ys[i] = h * (A32 * k[1][i]) + y[i];
  r = orc_rhs(p, t + C3 * h, ys, k[2]);
  (*nfe)++;
  if (r) return r;
  for (int i = 0; i < n; ++i) ys[i] = h * (A43 * k[2][i]) + y[i];
  r = orc_rhs(p, t + C4 * h, ys, k[3]);
  (*nfe)++;
  if (r) return r;
  for (int i = 0; i < n; ++i) {
    double s = A51 * k[0][i];
    s = s + A52 * k[1][i];
    s = s + A53 * k[2][i];
    s = s + A54 * k[3][i];
    ys[i] = h * s + y[i];
  }
  r = orc_rhs(p, t + C5 * h, ys, k[4]);
  (*nfe)++;
  if (r) return r;
  for (int i = 0; i < n; ++i) {
    double s = B1 * k[0][i];
    s = s + B2 * k[1][i];
    s = s + B3 * k[2][i];
    s = s + B4 * k[3][i];
    ynew[i] = h * s + y[i];
    double e = E1 * k[0][i];
    e = e + E2 * k[1][i];
    e = e + E3 * k[2][i];
    e = e + E4 * k[3][i];
    e = e + E5 * k[4][i];
    err[i] = h * e;
  }
  return 0;
}

static double wnorm(int n, const double *v, const double *w)
{
  return orc_wrms(n, v, w, 1);
}

int orc_integrate_erk(const orc_problem *p, const orc_opts *o, double t0, double tf, double *y, orc_stats *st)
{
  const int n = p->n;
  double ewt[ORC_NMAX], k1[ORC_NMAX], yn[ORC_NMAX], er[ORC_NMAX], tmp[ORC_NMAX], f1[ORC_NMAX];
  memset(st, 0, sizeof(*st));
  st->status = ORC_OK;
  st->q_last = 4;
  st->t_reached = t0;
  for (int i = 0; i < n; ++i)
    if (!isfinite(y[i])) { st->status = ORC_NONFINITE_INPUT; return st->status; }
  if (p->fext)
    for (int i = 0; i < n; ++i)
      if (!isfinite(p->fext[i])) { st->status = ORC_NONFINITE_INPUT; return st->status; }
  double t = t0;
  for (int i = 0; i < n; ++i) ewt[i] = 1.0 / (o->rtol * fabs(y[i]) + o->atol[i]);
  int r = orc_rhs(p, t, y, k1);
  st->nfe++;
  if (r) { st->status = ORC_RHS_FAIL; return st->status; }
  double h = o->h0;
  if (h == 0.0) {   /* Hairer-Wanner starting step */
    const double d0 = wnorm(n, y, ewt), d1 = wnorm(n, k1, ewt);
    double h0 = (d0 < 1e-5 || d1 < 1e-5) ? 1e-6 : 0.01 * (d0 / d1);
    if (h0 > tf - t0) h0 = tf - t0;
    for (int i = 0; i < n; ++i) tmp[i] = h0 * k1[i] + y[i];
    r = orc_rhs(p, t + h0, tmp, f1);
    st->nfe++;
    if (r < 0) { st->status = ORC_RHS_FAIL; return st->status; }
    if (r > 0) {
      h = h0;
    } else {
      for (int i = 0; i < n; ++i) tmp[i] = f1[i] - k1[i];
      const double d2 = wnorm(n, tmp, ewt) / h0;
      const double dm = fmax(d1, d2);
      const double h1 = (dm <= 1e-15) ? fmax(1e-6, h0 * 1e-3) : orc_root(0.01 / dm, 5);
      h = fmin(100.0 * h0, h1);
    }
  }
  if (h > tf - t0) h = tf - t0;
  if (o->hmax > 0.0 && h > o->hmax) h = o->hmax;
  double etamax = ERK_ETAMX1;
  for (;;) {
    if (st->nst >= o->mxstep) { st->status = ORC_TOO_MUCH_WORK; break; }
    /* one accepted step */
    int nef = 0, ncf = 0, have_k1 = 1, last = 0;
    double dsm = 0.0;
    for (;;) {
      last = 0;
      double hs = h;
      if ((t + hs - tf) >= 0.0) { hs = tf - t; last = 1; }
      int nfe = 0;
      r = orc_erk_step(p, t, hs, y, have_k1 ? k1 : NULL, yn, er, &nfe);
      st->nfe += nfe;
      have_k1 = 1;
      h = hs;
      if (r < 0) { st->status = ORC_RHS_FAIL; goto out; }
      if (r > 0) {                                    /* recoverable RHS failure: cut h */
        st->ncfn++;
        if (++ncf == ERK_MXNCF) { st->status = ORC_RHS_FAIL; goto out; }
        h = h * ERK_ETACF;
        etamax = 1.0;
        continue;
      }
      dsm = wnorm(n, er, ewt);
      if (dsm <= 1.0) break;
      st->netf++;
      if (++nef == ERK_MXNEF || fabs(h) <= o->hmin * (1.0 + ERK_UROUND)) { st->status = ORC_ERR_FAILURE; goto out; }
      double eta = ERK_SAFETY / sqrt(sqrt(dsm));
      eta = fmax(ERK_ETAMIN, eta);
      if (o->hmin > 0.0) eta = fmax(eta, o->hmin / fabs(h));
      h = h * eta;
      etamax = 1.0;
      if (t + h == t) { st->status = ORC_ERR_FAILURE; goto out; }
    }
    /* accept */
    st->nst++;
    t = last ? tf : t + h;
    for (int i = 0; i < n; ++i) y[i] = yn[i];
    st->h_last = h;
    if (last) break;
    double eta = (dsm == 0.0) ? etamax : ERK_SAFETY / sqrt(sqrt(dsm));
    eta = fmin(eta, etamax);
    if (o->hmax > 0.0) eta = fmin(eta, o->hmax / fabs(h));
    h = h * eta;
    etamax = ERK_ETAMX;
    for (int i = 0; i < n; ++i) ewt[i] = 1.0 / (o->rtol * fabs(y[i]) + o->atol[i]);
    r = orc_rhs(p, t, y, k1);
    st->nfe++;
    if (r) { st->status = ORC_RHS_FAIL; break; }
  }
out:
  st->t_reached = t;
  return st->status;
}
