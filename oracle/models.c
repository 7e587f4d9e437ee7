/*
 * models.c -- oracle right-hand sides and Jacobians (TEST INFRASTRUCTURE
 * ONLY; see oracle.h).  SURVEY.md §8(c).6.
 */
#include <complex.h>
#include <math.h>
#include <string.h>
#include "oracle.h"

/* ---- constant-volume reactor: real and complex instantiations --------- */
#define RT double
#define FN(x) x##_real
#define EXPF exp
#define LOGF log
#define REALPART(x) (x)
#include "mech_body.h"
#undef RT
#undef FN
#undef EXPF
#undef LOGF
#undef REALPART

#define RT double complex
#define FN(x) x##_cplx
#define EXPF cexp
#define LOGF clog
#define REALPART(x) creal(x)
#include "mech_body.h"
#undef RT
#undef FN
#undef EXPF
#undef LOGF
#undef REALPART

/* ---- Nyx-style heating/cooling (C2), reading R21, Appendix B ------------
 * State e [erg/g]; aux rho [g/cm^3].  Ionisation equilibrium (KWH96 eqs.
 * 33-38) solved for x_e = n_e/n_H by Illinois regula falsi on
 * [1e-12, 1+2 y_He], stop |dx_e| <= 1e-12 (1+2 y_He), <= 60 iterations,
 * every call from the same bracket (so R is a pure function of e).        */
typedef struct {
  double T, nH0, nHp, nHe0, nHep, nHepp, ne, g;
} kwh_pop;

static const double KWH_MP = 1.67262192369e-24;   /* g     */
static const double KWH_KB = 1.380649e-16;        /* erg/K */

static void kwh_eval(const orc_kwh_params *q, double e, double nH, double yHe,
                     double xe, kwh_pop *P)
{
  double mu = (1.0 + 4.0 * yHe) / (1.0 + yHe + xe);
  double T = (q->gamma_ad - 1.0) * mu * KWH_MP * e / KWH_KB;
  double sT = sqrt(T);
  double T3 = T / 1e3, T5 = T / 1e5, T6 = T / 1e6;
  double S5 = 1.0 / (1.0 + sqrt(T5));
  double aHp = 8.40e-11 / sT * pow(T3, -0.2) / (1.0 + pow(T6, 0.7));
  double aHep = 1.50e-10 * pow(T, -0.6353);
  double ad = 1.9e-3 * pow(T, -1.5) * exp(-470000.0 / T) * (1.0 + 0.3 * exp(-94000.0 / T));
  double aHepp = 3.36e-10 / sT * pow(T3, -0.2) / (1.0 + pow(T6, 0.7));
  double GeH0 = 5.85e-11 * sT * exp(-157809.1 / T) * S5;
  double GeHe0 = 2.38e-11 * sT * exp(-285335.4 / T) * S5;
  double GeHep = 5.68e-12 * sT * exp(-631515.0 / T) * S5;
  double ne = xe * nH;
  double nH0 = nH * aHp / (aHp + GeH0 + q->gph[0] / ne);
  double nHp = nH - nH0;
  double ion0 = GeHe0 + q->gph[1] / ne;      /* He0 -> He+  */
  double ion1 = GeHep + q->gph[2] / ne;      /* He+ -> He++ */
  double nHep = yHe * nH / (1.0 + (aHep + ad) / ion0 + ion1 / aHepp);
  double nHe0 = nHep * (aHep + ad) / ion0;
  double nHepp = nHep * ion1 / aHepp;
  double ne_new = nHp + nHep + 2.0 * nHepp;
  P->T = T; P->nH0 = nH0; P->nHp = nHp; P->nHe0 = nHe0; P->nHep = nHep;
  P->nHepp = nHepp; P->ne = ne; P->g = xe - ne_new / nH;
}

static int kwh_solve(const orc_problem *p, double e, kwh_pop *out);

static int kwh_rhs(const orc_problem *p, const double *y, double *f)
{
  kwh_pop Pp;
  if (kwh_solve(p, y[0], &Pp)) return 1;
  const kwh_pop *P = &Pp;
  const orc_kwh_params *q = p->kwh;
  double rho = p->rho;
  double T = P->T, sT = sqrt(T);
  double T3 = T / 1e3, T5 = T / 1e5, T6 = T / 1e6;
  double S5 = 1.0 / (1.0 + sqrt(T5));
  double ne = P->ne;
  double rec = pow(T3, -0.2) / (1.0 + pow(T6, 0.7));
  double L = 0.0;
  L += 7.50e-19 * exp(-118348.0 / T) * S5 * ne * P->nH0;
  L += 5.54e-17 * pow(T, -0.397) * exp(-473638.0 / T) * S5 * ne * P->nHep;
  L += 1.27e-21 * sT * exp(-157809.1 / T) * S5 * ne * P->nH0;
  L += 9.38e-22 * sT * exp(-285335.4 / T) * S5 * ne * P->nHe0;
  L += 4.95e-22 * sT * exp(-631515.0 / T) * S5 * ne * P->nHep;
  L += 8.70e-27 * sT * rec * ne * P->nHp;
  L += 1.55e-26 * pow(T, 0.3647) * ne * P->nHep;
  L += 3.48e-26 * sT * rec * ne * P->nHepp;
  L += 1.24e-13 * pow(T, -1.5) * exp(-470000.0 / T) * (1.0 + 0.3 * exp(-94000.0 / T)) * ne * P->nHep;
  double lt = 5.5 - log10(T);
  double gff = 1.1 + 0.34 * exp(-lt * lt / 3.0);
  L += 1.42e-27 * gff * sT * (P->nHp + P->nHep + 4.0 * P->nHepp) * ne;
  double zp1 = 1.0 + q->z;
  L += 5.41e-36 * ne * T * (zp1 * zp1 * zp1 * zp1);
  double H = P->nH0 * q->eph[0] + P->nHe0 * q->eph[1] + P->nHep * q->eph[2];
  f[0] = (H - L) / rho;
  if (p->fext) f[0] = f[0] + p->fext[0];
  return 0;
}

/* ionisation-equilibrium solve for x_e (shared by the RHS and the pin entry) */
static int kwh_solve(const orc_problem *p, double e, kwh_pop *out)
{
  const orc_kwh_params *q = p->kwh;
  double rho = p->rho;
  double nH = q->X * rho / KWH_MP;
  double yHe = q->Y / (4.0 * q->X);
  double xmax = 1.0 + 2.0 * yHe;
  if (!(e > 0.0) || !isfinite(e)) return 1;
  /* realisability (reading R17): T in [1, 1e9] K over the whole bracket */
  double Tmax = (q->gamma_ad - 1.0) * ((1.0 + 4.0 * yHe) / (1.0 + yHe + 1e-12)) * KWH_MP * e / KWH_KB;
  double Tmin = (q->gamma_ad - 1.0) * ((1.0 + 4.0 * yHe) / (1.0 + yHe + xmax)) * KWH_MP * e / KWH_KB;
  if (Tmin < 1.0 || Tmax > 1e9) return 1;

  kwh_pop A, B, Cc;
  double a = 1e-12, b = xmax;
  kwh_eval(q, e, nH, yHe, a, &A);
  kwh_eval(q, e, nH, yHe, b, &B);
  double fa = A.g, fb = B.g;
  kwh_pop *P;
  if (fb == 0.0) {
    P = &B;
  } else if (fa >= 0.0) {
    P = &A;
  } else {
    double tol = 1e-12 * xmax, cprev = 0.0;
    int side = 0;
    for (int it = 0; it < 60; ++it) {
      double c = (a * fb - b * fa) / (fb - fa);
      kwh_eval(q, e, nH, yHe, c, &Cc);
      double fc = Cc.g;
      if (it > 0 && fabs(c - cprev) <= tol) break;
      cprev = c;
      if (fc == 0.0) break;
      if ((fc > 0.0) == (fb > 0.0)) {
        b = c; fb = fc;
        if (side == -1) fa *= 0.5;
        side = -1;
      } else {
        a = c; fa = fc;
        if (side == +1) fb *= 0.5;
        side = +1;
      }
    }
    P = &Cc;
  }
  *out = *P;
  return 0;
}

/* pin entry: converged populations [T, nH0, nH+, nHe0, nHe+, nHe++, ne, g] */
int orc_kwh_state(const orc_problem *p, double e, double *out8)
{
  kwh_pop P;
  int r = kwh_solve(p, e, &P);
  out8[0] = P.T; out8[1] = P.nH0; out8[2] = P.nHp; out8[3] = P.nHe0;
  out8[4] = P.nHep; out8[5] = P.nHepp; out8[6] = P.ne; out8[7] = P.g;
  return r;
}

/* ---- RHS magnitude scale S_i (reading R19): the RHS evaluated with the
 * absolute value of every term, so that |f_gpu - f_orc| <= 1e-12 S is a
 * cancellation-proof parity criterion.               */
int orc_rhs_scale(const orc_problem *p, double t, const double *y, double *S)
{
  (void)t;
  int n = p->n;
  double f[ORC_NMAX];
  switch (p->kind) {
  case ORC_MODEL_LINEAR:
    for (int i = 0; i < n; ++i) S[i] = fabs(p->lambda[i] * y[i]) + (p->fext ? fabs(p->fext[i]) : 0.0);
    return 0;
  case ORC_MODEL_ROBERTSON: {
    const double *k = p->rob_k;
    double r1 = fabs(k[0] * y[0]), r2 = fabs(k[1] * y[1] * y[1]), r3 = fabs(k[2] * y[1] * y[2]);
    S[0] = r1 + r3; S[1] = r1 + r2 + r3; S[2] = r2;
    if (p->fext) for (int i = 0; i < 3; ++i) S[i] += fabs(p->fext[i]);
    return 0;
  }
  case ORC_MODEL_KWH: {
    /* heating + cooling magnitudes: |H| + |L| = |f - F| evaluated from both signs */
    orc_problem q = *p;
    q.fext = NULL;
    int r = kwh_rhs(&q, y, f);
    double e = fabs(f[0]);
    /* cooling and heating are each bounded by the sum of their terms; use
     * the heating-only and cooling-only parts from the populations */
    kwh_pop P;
    if (!r && !kwh_solve(p, y[0], &P)) {
      const orc_kwh_params *kp = p->kwh;
      double H = P.nH0 * kp->eph[0] + P.nHe0 * kp->eph[1] + P.nHep * kp->eph[2];
      e = fabs(H / p->rho) + fabs(H / p->rho - f[0]);
    }
    S[0] = e + (p->fext ? fabs(p->fext[0]) : 0.0);
    return r;
  }
  case ORC_MODEL_MECH:
    return mech_rhs_real(p, y, f, S);
  }
  return -1;
}

/* ---- dispatch ---------------------------------------------------------- */
int orc_rhs(const orc_problem *p, double t, const double *y, double *f)
{
  (void)t;
  int n = p->n;
  switch (p->kind) {
  case ORC_MODEL_LINEAR:
    /* f = lambda .* y + f_ext */
    for (int i = 0; i < n; ++i) {
      f[i] = p->lambda[i] * y[i];
      if (p->fext) f[i] = f[i] + p->fext[i];
    }
    return 0;
  case ORC_MODEL_ROBERTSON: {
    /* S:180; §8c.6 C1 */
    const double *k = p->rob_k;
    double r1 = k[0] * y[0], r2 = k[1] * y[1] * y[1], r3 = k[2] * y[1] * y[2];
    f[0] = -r1 + r3;
    f[1] = r1 - r3 - r2;
    f[2] = r2;
    if (p->fext) for (int i = 0; i < 3; ++i) f[i] = f[i] + p->fext[i];
    return 0;
  }
  case ORC_MODEL_KWH:
    return kwh_rhs(p, y, f);
  case ORC_MODEL_MECH:
    return mech_rhs_real(p, y, f, NULL);
  }
  return -1;
}

int orc_jac(const orc_problem *p, double t, const double *y, double *J)
{
  (void)t;
  int n = p->n;
  memset(J, 0, sizeof(double) * n * n);
  switch (p->kind) {
  case ORC_MODEL_LINEAR:
    for (int i = 0; i < n; ++i) J[i * n + i] = p->lambda[i];
    return 0;
  case ORC_MODEL_ROBERTSON: {
    const double *k = p->rob_k;
    J[0] = -k[0];            J[1] = k[2] * y[2];                       J[2] = k[2] * y[1];
    J[3] = k[0];             J[4] = -k[2] * y[2] - 2.0 * k[1] * y[1];  J[5] = -k[2] * y[1];
    J[6] = 0.0;              J[7] = 2.0 * k[1] * y[1];                 J[8] = 0.0;
    return 0;
  }
  case ORC_MODEL_MECH: {
    /* complex step: J[:,j] = Im f(y + i eps e_j) / eps, eps = 1e-30
     * (no subtractive cancellation; exact to rounding), §8c.4          */
    const double eps = 1e-30;
    double complex yc[ORC_NMAX], fc[ORC_NMAX];
    for (int j = 0; j < n; ++j) {
      for (int i = 0; i < n; ++i) yc[i] = y[i];
      yc[j] = y[j] + I * eps;
      int r = mech_rhs_cplx(p, yc, fc, NULL);
      if (r) return r;
      for (int i = 0; i < n; ++i) J[i * n + j] = cimag(fc[i]) / eps;
    }
    return 0;
  }
  }
  return -1;
}
