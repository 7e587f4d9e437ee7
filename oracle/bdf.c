/*
 * bdf.c -- oracle variable-order, variable-step BDF for ONE cell
 * (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * This is SURVEY.md §8(c).2 ("listing") written out in its own order: the
 * CVODE fixed-leading-coefficient Nordsieck BDF (orders 1..5) that the paper
 * uses with modified Newton and a
 * dense direct LU solver with pivoting or CVDiag.  Constants
 * are listing §8c.1 (paper-given: c_eps = 0.1, c_r = 0.3; all others
 * are CVODE defaults, paper silent).  Readings R1..R24 in DESIGN.md.
 *
 * Notation follows the listing: zn[j] = h^j y^(j)/j!, q order, L = q+1,
 * tau[1..6] past step sizes (most recent first), l[0..5], tq[1..5],
 * gamma = h/l[1], gammap = gamma at the last matrix setup, crate = R (Eq. 4).
 */
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

/* listing §8c.1 */
#define NLSCOEF 0.1     /* c_eps */
#define CRDOWN 0.3      /* c_r, */
#define MAXCOR 3
#define RDIV 2.0
#define MSBP 20
#define DGMAX 0.3
#define MSBJ 51
#define DGMAX_JBAD 0.2
#define BIAS1 6.0
#define BIAS2 6.0
#define BIAS3 10.0
#define ADDON 1e-6
#define THRESH 1.5
#define ETAMX1 1e4
#define ETAMX2 10.0
#define ETAMIN 0.1
#define ETAMXF 0.2
#define SMALL_NEF 2
#define MXNEF1 3
#define MXNEF 7
#define ETACF 0.25
#define MXNCF 10
#define LONG_WAIT 10
#define HUB_FACTOR 0.1
#define H_BIAS 0.5
#define HIN_ITERS 4
#define FRACT 0.1       /* CVDiag perturbation fraction */
#define UROUND DBL_EPSILON

enum { FIRST_CALL, PREV_CONV_FAIL, PREV_ERR_FAIL };
enum { CF_NONE, CF_BAD_J, CF_OTHER };
enum { NLS_OK = 0, NLS_RECOVERABLE = 1, NLS_RHS_UNREC = 2 };

/* storage of one cell (per-cell mode) */
typedef struct {
  double zn[ORC_QMAX + 1][ORC_NMAX];
  double ewt[ORC_NMAX], acor[ORC_NMAX], y[ORC_NMAX], ftemp[ORC_NMAX], tmp[ORC_NMAX];
  double ycor[ORC_NMAX], G[ORC_NMAX];
  double J[ORC_NMAX * ORC_NMAX], M[ORC_NMAX * ORC_NMAX];
  int piv[ORC_NMAX];
  double Minv[ORC_NMAX];
} cellbuf;

/* The integrator state.  Per-cell mode: one cell, nt = n.  Global-norm mode
 * (listing "Global-norm variant"; reading R14): the ncell cells of a
 * batch form ONE system of nt = n*ncell components (cell-major inside the
 * oracle), with one h, q and history; J is block diagonal (one n x n LU per
 * cell); every norm is batch-wide.                                          */
typedef struct {
  const orc_problem *p;
  const orc_opts *o;
  int n, qmax, global;
  long ncell, nt;
  const double *rho_all;           /* global: [ncell] */
  const double *fext_all;          /* global: [ncell][n] (cell-major) or NULL */
  double *zn[ORC_QMAX + 1];
  double *ewt, *acor, *y, *ftemp, *tmp, *ycor, *G;
  double *J, *M;                   /* [ncell][n][n] */
  int *piv;                        /* [ncell][n] */
  double *Minv;                    /* CVDiag */
  double gammasv;                  /* CVDiag */
  double tn, h, hscale, hprime, eta, etamax;
  double tau[ORC_QMAX + 2], l[ORC_QMAX + 1], tq[6];
  double rl1, gamma, gammap, gamrat, crate, acnrm, saved_tq5;
  int q, qprime, L, qwait;
  long nstlp, nstlj;
  orc_stats st;
} cell;

/*
 * x^(1/L) for the step-size factors (reading R25).  CVODE calls
 * libm's power function with exponent 1.0/L.  Here the real L-th root is
 * evaluated by a fixed sequence of IEEE operations that the GPU path
 * implements identically, so step-size decisions are bit-reproducible across
 * CPU and GPU:
 *   x = y 2^e, y in [1,2);  e = L k + r, 0 <= r < L;
 *   s ~ y^(-1/L): s0 = 1 - (y-1) c_L, then 4 Newton steps
 *       s <- s (1 + (1 - y s^L) / L)          (no division);
 *   x^(1/L) = ldexp(y s^(L-1) * 2^(r/L), k).
 * c_L = 1 - 2^(-1/L) and 2^(r/L) are correctly rounded constants.  The result
 * is within 12 ulp of the exact root (pinned in test_oracle_primitives.py).
 */
static const double ROOT_C[8][7] = {
  {0}, {1.0},
  {0x1.0p+0, 0x1.6a09e667f3bcdp+0},
  {0x1.0p+0, 0x1.428a2f98d728bp+0, 0x1.965fea53d6e3dp+0},
  {0x1.0p+0, 0x1.306fe0a31b715p+0, 0x1.6a09e667f3bcdp+0, 0x1.ae89f995ad3adp+0},
  {0x1.0p+0, 0x1.2611186bae675p+0, 0x1.51cb453b9536cp+0, 0x1.8406003b2ae5cp+0, 0x1.bdb8cdadbe120p+0},
  {0x1.0p+0, 0x1.1f59ac3c7d6c0p+0, 0x1.428a2f98d728bp+0, 0x1.6a09e667f3bcdp+0, 0x1.965fea53d6e3dp+0,
   0x1.c823e074ec129p+0},
  {0x1.0p+0, 0x1.1aa59c4115e7dp+0, 0x1.381147622f886p+0, 0x1.588cea3f093bep+0, 0x1.7c6a1f29e2ce6p+0,
   0x1.a402feeb9c533p+0, 0x1.cfbb031a741a5p+0}};
static const double ROOT_CL[8] = {0, 0, 0x1.2bec333018867p-2, 0x1.a68056b0a470ep-3, 0x1.45d819a94b14bp-3,
                                  0x1.091cc94907b7fp-3, 0x1.bee0fc589f6b6p-4, 0x1.8227e72c5f2dbp-4};

double orc_root(double x, int L)
{
  if (!(x > 0.0) || isinf(x)) return x > 0.0 ? x : 0.0;
  if (L == 1) return x;
  int e;
  double y = 2.0 * frexp(x, &e);              /* x = y 2^(e-1), y in [1, 2) */
  e = e - 1;
  int k = (e >= 0) ? e / L : -((-e + L - 1) / L);
  int r = e - L * k;                          /* 0 <= r < L */
  double invL = 1.0 / L;
  double s = 1.0 - (y - 1.0) * ROOT_CL[L];
  for (int it = 0; it < 4; ++it) {
    double p = s;
    for (int j = 0; j < L - 1; ++j) p = p * s;
    s = s * (1.0 + (1.0 - y * p) * invL);
  }
  double t = y;
  for (int j = 0; j < L - 1; ++j) t = t * s;
  return ldexp(t * ROOT_C[L][r], k);
}

/* x^(1/L) as the step-size controller uses it: plain mode (o->plain) calls
 * libm pow(x, 1.0/L) exactly as CVODE does; otherwise the fixed IEEE
 * sequence of reading R25 (bit-reproducible on the GPU). */
static double eta_root(int plain, double x, int L)
{
  return plain ? pow(x, 1.0 / L) : orc_root(x, L);
}

/* WRMS norm (Eq. 3).  Global mode: N = nt (reading R14) and the batch sum is
 * formed in a specified order (reading R15): per-cell sums in the group order,
 * accumulated sequentially over blocks of ORC_GBLK consecutive cells, block
 * partials accumulated sequentially.                                       */
static double wrms(cell *c, const double *v)
{
  if (!c->global) return orc_wrms(c->n, v, c->ewt, c->o->group);
  double S = 0.0;
  for (long b = 0; b < c->ncell; b += ORC_GBLK) {
    double P = 0.0;
    long e = b + ORC_GBLK < c->ncell ? b + ORC_GBLK : c->ncell;
    for (long k = b; k < e; ++k) P = P + orc_wrms_sum(c->n, v + k * c->n, c->ewt + k * c->n, c->o->group);
    S = S + P;
  }
  return sqrt(S / (double)c->nt);
}

/* Eq. 3 weights: w_i = 1/(rtol |y_i| + atol_i) */
static void set_ewt(cell *c, const double *y)
{
  for (long i = 0; i < c->nt; ++i) c->ewt[i] = 1.0 / (c->o->rtol * fabs(y[i]) + c->o->atol[i % c->n]);
}

static int f_eval(cell *c, double t, const double *y, double *f)
{
  c->st.nfe++;
  if (!c->global) return orc_rhs(c->p, t, y, f);
  int rv = 0;                      /* any cell's failure is the batch's (R18) */
  for (long k = 0; k < c->ncell; ++k) {
    orc_problem q = *c->p;
    q.rho = c->rho_all ? c->rho_all[k] : q.rho;
    q.fext = c->fext_all ? c->fext_all + k * c->n : NULL;
    int r = orc_rhs(&q, t, y + k * c->n, f + k * c->n);
    if (r < 0) return r;
    if (r > 0) rv = r;
  }
  return rv;
}

/* RESCALE: zn[j] *= eta^j; h = hscale*eta; hscale = h (cvRescale) */
static void rescale(cell *c)
{
  double r = c->eta;
  for (int j = 1; j <= c->q; ++j) {
    for (long i = 0; i < c->nt; ++i) c->zn[j][i] = r * c->zn[j][i];
    r = r * c->eta;
  }
  c->h = c->hscale * c->eta;
  c->hscale = c->h;
}

/* PREDICT: tn += h; Pascal-triangle update zn[j-1] += zn[j] (cvPredict) */
static void predict(cell *c, double tf)
{
  c->tn = c->tn + c->h;
  if ((c->tn - tf) * c->h > 0.0) c->tn = tf;          /* never pass tf (R11) */
  for (int k = 1; k <= c->q; ++k)
    for (int j = c->q; j >= k; --j)
      for (long i = 0; i < c->nt; ++i) c->zn[j - 1][i] = c->zn[j - 1][i] + c->zn[j][i];
}

/* RESTORE: undo PREDICT (cvRestore) */
static void restore(cell *c, double saved_t)
{
  c->tn = saved_t;
  for (int k = 1; k <= c->q; ++k)
    for (int j = c->q; j >= k; --j)
      for (long i = 0; i < c->nt; ++i) c->zn[j - 1][i] = c->zn[j - 1][i] - c->zn[j][i];
}

/* SET_BDF: cvSetBDF + cvSetTqBDF (listing) */
void orc_set_bdf(int q, double h, const double *tau, int qwait, double *l, double *tq)
{
  double xi_inv = 1.0, xistar_inv = 1.0, alpha0 = -1.0, alpha0_hat = -1.0, hsum = h;
  l[0] = l[1] = 1.0;
  for (int i = 2; i <= ORC_QMAX; ++i) l[i] = 0.0;
  if (q > 1) {
    for (int j = 2; j < q; ++j) {
      hsum = hsum + tau[j - 1];
      xi_inv = h / hsum;
      alpha0 = alpha0 - 1.0 / j;
      for (int i = j; i >= 1; --i) l[i] = l[i] + l[i - 1] * xi_inv;
    }
    alpha0 = alpha0 - 1.0 / q;
    xistar_inv = -l[1] - alpha0;
    hsum = hsum + tau[q - 1];
    xi_inv = h / hsum;
    alpha0_hat = -l[1] - xi_inv;
    for (int i = q; i >= 1; --i) l[i] = l[i] + l[i - 1] * xistar_inv;
  }
  /* cvSetTqBDF */
  double A1 = 1.0 - alpha0_hat + alpha0;
  double A2 = 1.0 + q * A1;
  tq[2] = fabs(A1 / (alpha0 * A2));
  tq[5] = fabs(A2 * xistar_inv / (l[q] * xi_inv));
  if (qwait == 1) {
    if (q > 1) {
      double C = xistar_inv / l[q];
      double A3 = alpha0 + 1.0 / q;
      double A4 = alpha0_hat + xi_inv;
      double Cpinv = (1.0 - A4 + A3) / A3;
      tq[1] = fabs(C * Cpinv);
    } else {
      tq[1] = 1.0;
    }
    hsum = hsum + tau[q];
    xi_inv = h / hsum;
    double A5 = alpha0 - 1.0 / (q + 1);
    double A6 = alpha0_hat - xi_inv;
    double Cppinv = (1.0 - A6 + A5) / A2;
    tq[3] = fabs(Cppinv / (xi_inv * (q + 2) * A5));
  }
  tq[4] = NLSCOEF / tq[2];            /* tol = c_eps * eps, eps = 1/tq[2] (R2) */
}

/* ADJUST_ORDER(+1): cvIncreaseBDF (hscale = old h, before RESCALE) */
static void increase_bdf(cell *c)
{
  double l[ORC_QMAX + 1];
  for (int i = 0; i <= ORC_QMAX; ++i) l[i] = 0.0;
  double alpha1 = 1.0, prod = 1.0, xiold = 1.0, alpha0 = -1.0, hsum = c->hscale;
  l[2] = 1.0;
  if (c->q > 1) {
    for (int j = 1; j < c->q; ++j) {
      hsum = hsum + c->tau[j + 1];
      double xi = hsum / c->hscale;
      prod = prod * xi;
      alpha0 = alpha0 - 1.0 / (j + 1);
      alpha1 = alpha1 + 1.0 / xi;
      for (int i = j + 2; i >= 2; --i) l[i] = l[i] * xiold + l[i - 1];
      xiold = xi;
    }
  }
  double A1 = (-alpha0 - alpha1) / prod;
  int Lq = c->q + 1;
  for (long i = 0; i < c->nt; ++i) c->zn[Lq][i] = A1 * c->zn[c->qmax][i];
  for (int j = 2; j <= c->q; ++j)
    for (long i = 0; i < c->nt; ++i) c->zn[j][i] = l[j] * c->zn[Lq][i] + c->zn[j][i];
}

/* ADJUST_ORDER(-1): cvDecreaseBDF */
static void decrease_bdf(cell *c)
{
  double l[ORC_QMAX + 1];
  for (int i = 0; i <= ORC_QMAX; ++i) l[i] = 0.0;
  l[2] = 1.0;
  double hsum = 0.0;
  for (int j = 1; j <= c->q - 2; ++j) {
    hsum = hsum + c->tau[j];
    double xi = hsum / c->hscale;
    for (int i = j + 2; i >= 2; --i) l[i] = l[i] * xi + l[i - 1];
  }
  for (int j = 2; j < c->q; ++j)
    for (long i = 0; i < c->nt; ++i) c->zn[j][i] = -l[j] * c->zn[c->q][i] + c->zn[j][i];
}

static void adjust_order(cell *c, int dq)
{
  if (c->q == 2 && dq != 1) return;   /* cvAdjustOrder: nothing to do 2 -> 1 */
  if (dq == 1) increase_bdf(c); else decrease_bdf(c);
}

/* residual G = (rl1 zn[1] + ycor) - gamma f(tn, zn[0] + ycor)  (cvNlsResidual) */
static int residual(cell *c, const double *ycor, double *G)
{
  for (long i = 0; i < c->nt; ++i) c->y[i] = c->zn[0][i] + ycor[i];
  int r = f_eval(c, c->tn, c->y, c->ftemp);
  if (r) return r;
  for (long i = 0; i < c->nt; ++i) {
    double t = c->rl1 * c->zn[1][i] + ycor[i];
    G[i] = -c->gamma * c->ftemp[i] + t;
  }
  return 0;
}

/* matrix setup (cvLsSetup dense / CVDiagSetup).  Returns 0, >0 recoverable,
 * <0 unrecoverable.  *jcur set when J was (re)evaluated.                  */
/* cvLsDenseDQJac (CVODE; the paper's finite-difference Jacobian, approaches 3A/3B) */
int orc_jac_dq(const orc_problem *p, double t, const double *y, const double *fy, const double *ewt, double h,
               double *J)
{
  const int n = p->n;
  const double srur = sqrt(UROUND);
  const double fnorm = orc_wrms(n, fy, ewt, 1);
  const double minInc = (fnorm != 0.0) ? (1000.0 * fabs(h) * UROUND * n * fnorm) : 1.0;
  double yp[ORC_NMAX], ft[ORC_NMAX];
  for (int i = 0; i < n; ++i) yp[i] = y[i];
  for (int j = 0; j < n; ++j) {
    const double yj = yp[j];
    const double inc = fmax(srur * fabs(yj), minInc / ewt[j]);
    yp[j] = yj + inc;
    const int r = orc_rhs(p, t, yp, ft);
    yp[j] = yj;
    if (r) return r;
    const double inc_inv = 1.0 / inc;
    for (int i = 0; i < n; ++i) J[i * n + j] = inc_inv * ft[i] + (-inc_inv) * fy[i];
  }
  return 0;
}

static int lsetup(cell *c, int convfail, int *jcur)
{
  int n = c->n;
  int rv = 0;
  if (c->o->ls == ORC_LS_DENSE || c->o->ls == ORC_LS_DENSE_DQ) {
    double dgamma = fabs(c->gamma / c->gammap - 1.0);
    int jbad = (c->st.nst == 0) || (c->st.nst >= c->nstlj + MSBJ) ||
               (convfail == CF_BAD_J && dgamma < DGMAX_JBAD) || (convfail == CF_OTHER);
    if (jbad) {
      c->st.nje++;
      c->nstlj = c->st.nst;
      *jcur = 1;
      for (long k = 0; k < c->ncell && rv == 0; ++k) {     /* block-diagonal J */
        orc_problem q = *c->p;
        if (c->global) {
          q.rho = c->rho_all ? c->rho_all[k] : q.rho;
          q.fext = c->fext_all ? c->fext_all + k * n : NULL;
        }
        if (c->o->ls == ORC_LS_DENSE_DQ) {   /* per-cell mode only (the global variant uses the analytic J) */
          const int r = orc_jac_dq(&q, c->tn, c->y + k * n, c->ftemp + k * n, c->ewt + k * n, c->h,
                                   c->J + k * n * n);
          if (r) rv = r > 0 ? 1 : -1;
        } else if (orc_jac(&q, c->tn, c->y + k * n, c->J + k * n * n)) {
          rv = -1;
        }
      }
    } else {
      *jcur = 0;
    }
    if (rv == 0) {
      for (long k = 0; k < c->ncell; ++k) {
        double *Mk = c->M + k * n * n;
        const double *Jk = c->J + k * n * n;
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j)
            Mk[i * n + j] = (i == j ? 1.0 : 0.0) - c->gamma * Jk[i * n + j];
        if (orc_lu_factor(n, Mk, c->piv + k * n)) rv = 1;   /* zero pivot: recoverable (R18) */
      }
    }
  } else {
    /* CVDiagSetup: diagonal difference-quotient J, M = I - gamma J */
    double r = FRACT * c->rl1;
    double yp[ORC_NMAX], fp[ORC_NMAX], ft[ORC_NMAX];
    for (int i = 0; i < n; ++i) ft[i] = c->h * c->ftemp[i] - c->zn[1][i];
    for (int i = 0; i < n; ++i) yp[i] = r * ft[i] + c->y[i];
    int fr = f_eval(c, c->tn, yp, fp);
    c->st.nje++;
    *jcur = 1;
    if (fr) {
      rv = fr;
    } else {
      for (int i = 0; i < n; ++i) {
        double Mi;
        if (fabs(ft[i] * c->ewt[i]) >= UROUND)
          Mi = (FRACT * ft[i] + (-c->h) * (fp[i] - c->ftemp[i])) / (FRACT * ft[i]);
        else
          Mi = 1.0;
        if (Mi == 0.0) { rv = 1; break; }
        c->Minv[i] = 1.0 / Mi;
      }
      c->gammasv = c->gamma;
    }
  }
  /* cvNlsLSetup bookkeeping */
  c->st.nsetups++;
  c->gamrat = 1.0;
  c->gammap = c->gamma;
  c->crate = 1.0;
  c->nstlp = c->st.nst;
  return rv;
}

/* Inexact Newton-Krylov (approaches 1A/1B; reading R29): A v = v - gamma Jv with the
 * difference-quotient Jv at the current Newton iterate y = zn0 + ycor (c->y) and fy = f(y) (c->ftemp):
 * sigma = 1/||v||_WRMS, Jv = (f(y + sigma v) - fy) (1/sigma), at most 3 tries with sigma *= 1/4 after a
 * recoverable RHS failure (CVODE cvLsDQJtimes); these RHS calls are not counted in nfe. */
#define EPLIFAC 0.05     /* c_l of Eq. 6 */
#define MAX_DQITERS 3
static int atimes_dq(void *ctx, const double *v, double *z)
{
  cell *c = (cell *)ctx;
  const int n = c->n;
  double w[ORC_NMAX], fw[ORC_NMAX];
  double sig = 1.0 / orc_wrms(n, v, c->ewt, c->o->group);
  int r = 0;
  for (int it = 0; it < MAX_DQITERS; ++it) {
    for (int i = 0; i < n; ++i) w[i] = sig * v[i] + c->y[i];
    r = orc_rhs(c->p, c->tn, w, fw);
    if (r == 0) break;
    if (r < 0) return -1;
    sig = sig * 0.25;
  }
  if (r > 0) return 1;
  const double siginv = 1.0 / sig;
  for (int i = 0; i < n; ++i) {
    const double jv = (fw[i] - c->ftemp[i]) * siginv;
    z[i] = v[i] - c->gamma * jv;
  }
  return 0;
}

/* cvLsSolve, iterative branch: if ||b||_WRMS <= deltar = c_l tq[4] return x = b (first Newton iteration)
 * or 0; else GMRES on the Eq. 5 system with S1 = S2 = diag(ewt) to the 2-norm tolerance deltar sqrt(n)
 * (Eq. 6); RES_REDUCED is accepted on the first Newton iteration only; every other failure is recoverable. */
static int lsolve_gmres(cell *c, double *b, int m)
{
  const int n = c->n;
  const double deltar = EPLIFAC * c->tq[4];
  const double bnorm = orc_wrms(n, b, c->ewt, c->o->group);
  if (bnorm <= deltar) {
    if (m > 0)
      for (int i = 0; i < n; ++i) b[i] = 0.0;
    return 0;
  }
  double ones = 0.0;
  for (int i = 0; i < n; ++i) ones = ones + 1.0 * 1.0;
  const double delta = deltar * sqrt(ones);
  double x[ORC_NMAX], rn;
  int nli = 0;
  const int maxl = c->o->maxl > 0 ? c->o->maxl : 5;
  const int r = orc_gmres(n, maxl, atimes_dq, c, b, c->ewt, c->ewt, delta, x, &nli, &rn);
  c->st.nli += nli;
  if (r == ORC_GMRES_ATIMES_FAIL_UNREC) return -1;
  if (r == ORC_GMRES_SUCCESS || (r == ORC_GMRES_RES_REDUCED && m == 0)) {
    for (int i = 0; i < n; ++i) b[i] = x[i];
    return 0;
  }
  return 1;
}

/* linear solve b <- M^{-1} b  (cvLsSolve dense with 2/(1+gamrat) / CVDiagSolve / GMRES); m = Newton iteration */
static int lsolve(cell *c, double *b, int m)
{
  int n = c->n;
  if (c->o->ls == ORC_LS_GMRES) return lsolve_gmres(c, b, m);
  if (c->o->ls != ORC_LS_DIAG) {
    for (long k = 0; k < c->ncell; ++k) {
      if (c->o->plain) orc_lu_solve_div(n, c->M + k * n * n, c->piv + k * n, b + k * n);
      else orc_lu_solve(n, c->M + k * n * n, c->piv + k * n, b + k * n);
    }
    if (c->gamrat != 1.0) {
      double s = 2.0 / (1.0 + c->gamrat);
      for (long i = 0; i < c->nt; ++i) b[i] = s * b[i];
    }
    return 0;
  }
  if (c->gammasv != c->gamma) {
    double r = c->gamma / c->gammasv;
    for (int i = 0; i < n; ++i) {
      double Mi = (1.0 / c->Minv[i] + (-1.0)) * r + 1.0;
      if (Mi == 0.0) return 1;
      c->Minv[i] = 1.0 / Mi;
    }
    c->gammasv = c->gamma;
  }
  for (int i = 0; i < n; ++i) b[i] = b[i] * c->Minv[i];
  return 0;
}

/* NEWTON(nflag): cvNls + SUNNonlinSol_Newton + cvNlsConvTest (Eq. 4) */
static int newton(cell *c, int nflag)
{
  long n = c->nt;
  int convfail = (nflag == FIRST_CALL || nflag == PREV_ERR_FAIL) ? CF_NONE : CF_OTHER;
  int setup = (nflag == PREV_CONV_FAIL) || (nflag == PREV_ERR_FAIL) || (c->st.nst == 0) ||
              (c->st.nst >= c->nstlp + MSBP) || (fabs(c->gamrat - 1.0) > DGMAX);
  /* matrix-free GMRES without a preconditioner has no setup (CVODE sets lsetup = NULL): R = 1 at every
   * solve, no matrix refresh and no retry after a failure (reading R29) */
  const int msetup = c->o->ls != ORC_LS_GMRES;
  if (!msetup) {
    setup = 0;
    c->crate = 1.0;
  }
  double *ycor = c->ycor, *G = c->G;
  double tol = c->tq[4];
  int jcur = 0;
  for (long i = 0; i < n; ++i) ycor[i] = 0.0;
  for (;;) {
    int rv = residual(c, ycor, G);                               /* N4 */
    if (rv < 0) return NLS_RHS_UNREC;
    /* a failed first residual (of the solve or of its retry) is not retried: SUNNonlinSol_Newton leaves its
     * loop before the retry logic (reading R5; retrying would re-evaluate the same failing state forever) */
    if (rv > 0) return NLS_RECOVERABLE;
    if (rv == 0 && setup) {
      rv = lsetup(c, convfail, &jcur);
      if (rv < 0) return NLS_RHS_UNREC;
      setup = 0;
    }
    if (rv == 0) {
      double dprev = 0.0;
      int m = 0;
      for (;;) {                                                  /* N6 */
        c->st.nni++;
        for (long i = 0; i < n; ++i) G[i] = -G[i];
        rv = lsolve(c, G, m);
        if (rv < 0) return NLS_RHS_UNREC;
        if (rv) break;
        for (long i = 0; i < n; ++i) ycor[i] = ycor[i] + G[i];
        double del = wrms(c, G);
        if (m > 0) c->crate = fmax(CRDOWN * c->crate, del / dprev);     /* Eq. 4 rate */
        double dcon = del * fmin(1.0, c->crate) / tol;
        if (dcon <= 1.0) {                                                /* Eq. 4 test */
          c->acnrm = (m == 0) ? del : wrms(c, ycor);
          for (long i = 0; i < n; ++i) c->acor[i] = ycor[i];
          return NLS_OK;
        }
        if (m >= 1 && del > RDIV * dprev) { rv = 1; break; }
        dprev = del;
        m++;
        if (m >= MAXCOR) { rv = 1; break; }
        rv = residual(c, ycor, G);
        if (rv < 0) return NLS_RHS_UNREC;
        if (rv) break;
      }
    }
    /* FAIL: retry once with a fresh Jacobian if it was not current */
    if (rv > 0 && !jcur && msetup) {
      setup = 1;
      convfail = CF_BAD_J;
      for (long i = 0; i < n; ++i) ycor[i] = 0.0;
      continue;
    }
    return NLS_RECOVERABLE;
  }
}

/* SET_ETA (cvSetEta): eta < THRESH keeps h; else cap by etamax and hmax */
static double set_eta_scalar(double eta, double etamax, double h, double hmax, double *hprime)
{
  if (eta < THRESH) {
    *hprime = h;
    return 1.0;
  }
  eta = fmin(eta, etamax);
  if (hmax > 0.0) eta = eta / fmax(1.0, fabs(h) * eta / hmax);
  *hprime = h * eta;
  return eta;
}

/* PREPARE_NEXT scalar part (cvPrepareNextStep + cvChooseEta + cvSetEta),
 * exported for the controller pins.  in/out *qwait; dsm = ||LTE|| at order q;
 * ddn = ||zn[q]|| tq[1] (used iff q > 1), dup = ||acor - c zn[qmax]|| tq[3]
 * (used iff have_up); both only consulted when *qwait == 0.  Returns eta,
 * sets *qprime and *hprime.  Tie-break (reading R8): q, then q-1, then q+1. */
double orc_choose_eta(int q, int *qwait, double etamax, double h, double hmax, double dsm, double ddn,
                      int have_up, double dup, int plain, int *qprime, double *hprime)
{
  const int L = q + 1;
  if (etamax == 1.0) {
    *qwait = *qwait > 2 ? *qwait : 2;
    *qprime = q;
    *hprime = h;
    return 1.0;
  }
  double etaq = 1.0 / (eta_root(plain, BIAS2 * dsm, L) + ADDON);
  if (*qwait != 0) {
    *qprime = q;
    return set_eta_scalar(etaq, etamax, h, hmax, hprime);
  }
  *qwait = 2;
  double etaqm1 = 0.0, etaqp1 = 0.0;
  if (q > 1) etaqm1 = 1.0 / (eta_root(plain, BIAS1 * ddn, q) + ADDON);
  if (have_up) etaqp1 = 1.0 / (eta_root(plain, BIAS3 * dup, L + 1) + ADDON);
  double etam = fmax(etaqm1, fmax(etaq, etaqp1));
  double eta;
  if (etam < THRESH) {
    eta = 1.0;
    *qprime = q;
  } else if (etam == etaq) {
    eta = etaq;
    *qprime = q;
  } else if (etam == etaqm1) {
    eta = etaqm1;
    *qprime = q - 1;
  } else {
    eta = etaqp1;
    *qprime = q + 1;
  }
  return set_eta_scalar(eta, etamax, h, hmax, hprime);
}

/* PREPARE_NEXT (cvPrepareNextStep + cvChooseEta): the two extra norms, then
 * the scalar choice above; zn[qmax] = acor when the order is raised. */
static void prepare_next(cell *c, double dsm)
{
  long n = c->nt;
  double ddn = 0.0, dup = 0.0;
  int have_up = 0;
  if (c->etamax != 1.0 && c->qwait == 0) {
    if (c->q > 1) ddn = wrms(c, c->zn[c->q]) * c->tq[1];
    if (c->q != c->qmax && c->saved_tq5 != 0.0) {
      double hr = c->h / c->tau[2];
      double pw = 1.0;
      for (int k = 0; k < c->L; ++k) pw = pw * hr;
      double cquot = (c->tq[5] / c->saved_tq5) * pw;
      for (long i = 0; i < n; ++i) c->tmp[i] = -cquot * c->zn[c->qmax][i] + c->acor[i];
      dup = wrms(c, c->tmp) * c->tq[3];
      have_up = 1;
    }
  }
  int q0 = c->q;
  c->eta = orc_choose_eta(c->q, &c->qwait, c->etamax, c->h, c->o->hmax, dsm, ddn, have_up, dup, c->o->plain,
                          &c->qprime, &c->hprime);
  if (c->qprime == q0 + 1)
    for (long i = 0; i < n; ++i) c->zn[c->qmax][i] = c->acor[i];
}

/* cvHin: initial step estimate (reading R9) */
static int hin(cell *c, double t0, double tf, double *h0)
{
  long n = c->nt;
  double tdist = tf - t0;
  double tround = UROUND * fmax(fabs(t0), fabs(tf));
  double hlb = 100.0 * tround;
  /* cvUpperBoundH0 */
  double hub_inv = 0.0;
  for (long i = 0; i < n; ++i) {
    double d = HUB_FACTOR * fabs(c->zn[0][i]) + 1.0 / c->ewt[i];
    double r = fabs(c->zn[1][i]) / d;
    if (r > hub_inv) hub_inv = r;
  }
  double hub = HUB_FACTOR * tdist;
  if (hub * hub_inv > 1.0) hub = 1.0 / hub_inv;
  double hg = sqrt(hlb * hub);
  if (hub < hlb) { *h0 = hg; return 0; }
  double hs = hg, hnew = hg;
  for (int count1 = 1; count1 <= HIN_ITERS; ++count1) {
    int ok = 0;
    double yddnrm = 0.0;
    for (int count2 = 1; count2 <= HIN_ITERS; ++count2) {
      /* cvYddNorm: ydd = (f(t0+hg, y0 + hg f0) - f0) * (1/hg) */
      double *yt = c->ycor, *ft = c->G;     /* scratch (not yet in use) */
      for (long i = 0; i < n; ++i) yt[i] = hg * c->zn[1][i] + c->zn[0][i];
      int r = f_eval(c, t0 + hg, yt, ft);
      if (r < 0) return -1;
      if (r == 0) {
        double ih = 1.0 / hg;
        for (long i = 0; i < n; ++i) ft[i] = (ft[i] - c->zn[1][i]) * ih;
        yddnrm = wrms(c, ft);
        ok = 1;
        break;
      }
      hg = hg * 0.2;
    }
    if (!ok) {
      if (count1 <= 2) return -1;
      hnew = hs;
      break;
    }
    hs = hg;
    hnew = (yddnrm * hub * hub > 2.0) ? sqrt(2.0 / yddnrm) : sqrt(hg * hub);
    if (count1 == HIN_ITERS) break;
    double hrat = hnew / hg;
    if (hrat > 0.5 && hrat < 2.0) break;
    if (count1 > 1 && hrat > 2.0) { hnew = hg; break; }
    hg = hnew;
  }
  double h = H_BIAS * hnew;
  if (h < hlb) h = hlb;
  if (h > hub) h = hub;
  *h0 = h;
  return 0;
}

/* STEP: one accepted step of cvStep.  Returns ORC_OK or a failure status. */
static int step(cell *c, double tf)
{
  long n = c->nt;
  double saved_t = c->tn;
  int ncf = 0, nef = 0, nflag = FIRST_CALL;
  if (c->st.nst > 0 && c->hprime != c->h) {
    if (c->qprime != c->q) {
      adjust_order(c, c->qprime - c->q);
      c->q = c->qprime;
      c->L = c->q + 1;
      c->qwait = c->L;
    }
    rescale(c);
  }
  double dsm;
  for (;;) {
    predict(c, tf);
    orc_set_bdf(c->q, c->h, c->tau, c->qwait, c->l, c->tq);
    c->rl1 = 1.0 / c->l[1];
    c->gamma = c->h * c->rl1;
    if (c->st.nst == 0) c->gammap = c->gamma;
    c->gamrat = (c->st.nst > 0) ? c->gamma / c->gammap : 1.0;

    int r = newton(c, nflag);
    if (r != NLS_OK) {
      /* cvHandleNFlag: convergence failure */
      c->st.ncfn++;
      restore(c, saved_t);
      if (r == NLS_RHS_UNREC) return ORC_RHS_FAIL;
      ncf++;
      c->etamax = 1.0;
      if (fabs(c->h) <= c->o->hmin * (1.0 + UROUND) || ncf == MXNCF) return ORC_CONV_FAILURE;
      c->eta = fmax(ETACF, c->o->hmin / fabs(c->h));
      nflag = PREV_CONV_FAIL;
      rescale(c);
      continue;
    }
    /* local error test, ||LTE|| = acnrm * tq[2] <= 1 */
    dsm = c->acnrm * c->tq[2];
    if (dsm <= 1.0) break;
    nef++;
    c->st.netf++;
    nflag = PREV_ERR_FAIL;
    restore(c, saved_t);
    if (fabs(c->h) <= c->o->hmin * (1.0 + UROUND) || nef == MXNEF) return ORC_ERR_FAILURE;
    c->etamax = 1.0;
    if (nef <= MXNEF1) {
      c->eta = 1.0 / (eta_root(c->o->plain, BIAS2 * dsm, c->L) + ADDON);
      c->eta = fmax(ETAMIN, fmax(c->eta, c->o->hmin / fabs(c->h)));
      if (nef >= SMALL_NEF) c->eta = fmin(c->eta, ETAMXF);
      rescale(c);
      continue;
    }
    if (c->q > 1) {
      c->eta = fmax(ETAMIN, c->o->hmin / fabs(c->h));
      adjust_order(c, -1);
      c->L = c->q;
      c->q = c->q - 1;
      c->qwait = c->L;
      rescale(c);
      continue;
    }
    c->eta = fmax(ETAMIN, c->o->hmin / fabs(c->h));
    c->h = c->h * c->eta;
    c->hprime = c->h;
    c->hscale = c->h;
    c->qwait = LONG_WAIT;
    int fr = f_eval(c, c->tn, c->zn[0], c->tmp);
    if (fr < 0) return ORC_RHS_FAIL;
    if (fr > 0) return ORC_RHS_FAIL;
    for (long i = 0; i < n; ++i) c->zn[1][i] = c->h * c->tmp[i];
  }

  /* DONE: cvCompleteStep */
  c->st.nst++;
  for (int i = c->q; i >= 2; --i) c->tau[i] = c->tau[i - 1];
  if (c->q == 1 && c->st.nst > 1) c->tau[2] = c->tau[1];
  c->tau[1] = c->h;
  for (int j = 0; j <= c->q; ++j)
    for (long i = 0; i < n; ++i) c->zn[j][i] = c->l[j] * c->acor[i] + c->zn[j][i];
  c->qwait--;
  if (c->qwait == 1 && c->q != c->qmax) {
    for (long i = 0; i < n; ++i) c->zn[c->qmax][i] = c->acor[i];
    c->saved_tq5 = c->tq[5];
  }
  prepare_next(c, dsm);
  c->etamax = ETAMX2;
  return ORC_OK;
}

/* INIT + LOOP (O1-O5) on an initialised cell c; y: [nt] in/out */
static void run(cell *c, double t0, double tf, double *y, orc_trace *tr)
{
  const orc_opts *o = c->o;
  long n = c->nt;
  c->st.status = ORC_OK;
  c->st.t_reached = t0;
  for (long i = 0; i < n; ++i)
    if (!isfinite(y[i])) { c->st.status = ORC_NONFINITE_INPUT; goto out; }
  if (!c->global && c->p->fext) {
    for (int i = 0; i < c->n; ++i)
      if (!isfinite(c->p->fext[i])) { c->st.status = ORC_NONFINITE_INPUT; goto out; }
  }
  if (c->global && c->fext_all) {
    for (long i = 0; i < n; ++i)
      if (!isfinite(c->fext_all[i])) { c->st.status = ORC_NONFINITE_INPUT; goto out; }
  }

  /* INIT */
  for (long i = 0; i < n; ++i) c->zn[0][i] = y[i];
  set_ewt(c, y);
  c->tn = t0;
  if (f_eval(c, t0, y, c->zn[1])) { c->st.status = ORC_RHS_FAIL; goto out; }
  double h0 = o->h0;
  if (h0 == 0.0) {
    if (hin(c, t0, tf, &h0)) { c->st.status = ORC_RHS_FAIL; goto out; }
  }
  if (h0 > tf - t0) h0 = tf - t0;
  if (o->hmax > 0.0 && h0 > o->hmax) h0 = o->hmax;
  for (long i = 0; i < n; ++i) c->zn[1][i] = h0 * c->zn[1][i];
  c->h = c->hscale = c->hprime = h0;
  c->q = c->qprime = 1;
  c->L = 2;
  c->qwait = 2;
  c->etamax = ETAMX1;
  c->crate = 1.0;
  c->eta = 1.0;

  /* LOOP */
  for (;;) {
    if (c->st.nst > 0) set_ewt(c, c->zn[0]);                        /* O1 */
    if ((c->tn + c->hprime - tf) * c->h > 0.0) {                     /* O2 */
      c->hprime = tf - c->tn;
      c->eta = c->hprime / c->h;
    }
    if (c->st.nst >= o->mxstep) { c->st.status = ORC_TOO_MUCH_WORK; break; }   /* O3 */
    int r = step(c, tf);                                             /* O4 */
    if (r != ORC_OK) { c->st.status = r; break; }
    if (tr && tr->count < tr->cap) {
      int k = tr->count++;
      tr->tn[k] = c->tn; tr->h[k] = c->h; tr->q[k] = c->q;
      for (int j = 0; j <= ORC_QMAX; ++j)
        for (long i = 0; i < n; ++i) tr->zn[(k * (ORC_QMAX + 1) + j) * n + i] = c->zn[j][i];
    }
    if (fabs(c->tn - tf) <= 100.0 * UROUND * (fabs(c->tn) + fabs(c->h))) {   /* O5 */
      c->tn = tf;
      break;
    }
  }
  for (long i = 0; i < n; ++i) y[i] = c->zn[0][i];
  c->st.t_reached = c->tn;
out:
  c->st.q_last = c->q;
  c->st.h_last = c->h;
}

int orc_integrate(const orc_problem *p, const orc_opts *o, double t0, double tf,
                  double *y, orc_stats *st, orc_trace *tr)
{
  if (o->method == ORC_METHOD_ERK4) return orc_integrate_erk(p, o, t0, tf, y, st);
  cellbuf B;
  cell C;
  cell *c = &C;
  memset(c, 0, sizeof(*c));
  memset(&B, 0, sizeof(B));
  c->p = p; c->o = o; c->n = p->n;
  c->ncell = 1; c->nt = p->n; c->global = 0;
  c->qmax = o->qmax < 1 ? 1 : (o->qmax > ORC_QMAX ? ORC_QMAX : o->qmax);
  for (int j = 0; j <= ORC_QMAX; ++j) c->zn[j] = B.zn[j];
  c->ewt = B.ewt; c->acor = B.acor; c->y = B.y; c->ftemp = B.ftemp; c->tmp = B.tmp;
  c->ycor = B.ycor; c->G = B.G; c->J = B.J; c->M = B.M; c->piv = B.piv; c->Minv = B.Minv;
  run(c, t0, tf, y, tr);
  *st = c->st;
  return c->st.status;
}

/* One NEWTON solve of the listing on a given predicted state, for the
 * Newton replay pin: nst = 0, so the matrix is set up and J
 * evaluated at y = zn0 (ycor = 0), gamma = h rl1, gamrat = 1, R = 1,
 * tol = the caller's (tq[4]).  Outputs acor (= ycor at convergence), acnrm,
 * the number of Newton iterations and RHS evaluations.  Returns 0 (converged),
 * 1 (recoverable failure) or 2 (unrecoverable RHS failure).               */
int orc_newton_once(const orc_problem *p, const orc_opts *o, double tn, double h, double rl1, double tol,
                    const double *zn0, const double *zn1, const double *ewt, double *acor, double *acnrm,
                    int *nni, int *nfe)
{
  cellbuf B;
  cell C;
  cell *c = &C;
  memset(c, 0, sizeof(*c));
  memset(&B, 0, sizeof(B));
  c->p = p; c->o = o; c->n = p->n;
  c->ncell = 1; c->nt = p->n; c->global = 0;
  c->qmax = ORC_QMAX;
  for (int j = 0; j <= ORC_QMAX; ++j) c->zn[j] = B.zn[j];
  c->ewt = B.ewt; c->acor = B.acor; c->y = B.y; c->ftemp = B.ftemp; c->tmp = B.tmp;
  c->ycor = B.ycor; c->G = B.G; c->J = B.J; c->M = B.M; c->piv = B.piv; c->Minv = B.Minv;
  for (int i = 0; i < c->n; ++i) {
    c->zn[0][i] = zn0[i];
    c->zn[1][i] = zn1[i];
    c->ewt[i] = ewt[i];
  }
  c->tn = tn;
  c->h = h;
  c->q = 1;
  c->rl1 = rl1;
  c->gamma = h * rl1;
  c->gammap = c->gamma;
  c->gamrat = 1.0;
  c->crate = 1.0;
  c->tq[4] = tol;
  int r = newton(c, FIRST_CALL);
  for (int i = 0; i < c->n; ++i) acor[i] = c->acor[i];
  *acnrm = c->acnrm;
  *nni = c->st.nni;
  *nfe = c->st.nfe;
  return r;
}

/* Global-norm mode (listing "Global-norm variant"): the N cells
 * of a YC field y[k*N + c] integrated as ONE system -- one h, q, history and
 * batch-wide WRMS norms (N_tot = n*N, reading R14); block-diagonal J with one
 * LU per cell; any cell's zero pivot or RHS failure is the batch's
 * recoverable failure (R18).  Dense solver only.                          */
int orc_integrate_global(const orc_problem *proto, const orc_opts *o, double t0, double tf, int64_t N,
                         double *y, const double *fext, const double *rho, orc_stats *st)
{
  int n = proto->n;
  long nt = (long)n * N;
  cell C;
  cell *c = &C;
  memset(c, 0, sizeof(*c));
  c->p = proto; c->o = o; c->n = n;
  c->ncell = N; c->nt = nt; c->global = 1;
  c->qmax = o->qmax < 1 ? 1 : (o->qmax > ORC_QMAX ? ORC_QMAX : o->qmax);
  double *mem = calloc((size_t)nt * (ORC_QMAX + 1 + 7) + (size_t)nt * n * 2 + (fext ? nt : 0), sizeof(double));
  int *piv = calloc((size_t)nt, sizeof(int));
  double *ycm = calloc((size_t)nt, sizeof(double));
  if (!mem || !piv || !ycm) { free(mem); free(piv); free(ycm); return -1; }
  double *q = mem;
  for (int j = 0; j <= ORC_QMAX; ++j) { c->zn[j] = q; q += nt; }
  c->ewt = q; q += nt; c->acor = q; q += nt; c->y = q; q += nt; c->ftemp = q; q += nt;
  c->tmp = q; q += nt; c->ycor = q; q += nt; c->G = q; q += nt;
  c->J = q; q += nt * n; c->M = q; q += nt * n;
  double *fcm = NULL;
  if (fext) { fcm = q; q += nt; }
  c->piv = piv;
  c->Minv = NULL;
  c->rho_all = rho;
  /* YC -> cell-major */
  for (long k = 0; k < N; ++k)
    for (int i = 0; i < n; ++i) {
      ycm[k * n + i] = y[(long)i * N + k];
      if (fext) fcm[k * n + i] = fext[(long)i * N + k];
    }
  c->fext_all = fcm;
  run(c, t0, tf, ycm, NULL);
  if (c->st.status != ORC_NONFINITE_INPUT)
    for (long k = 0; k < N; ++k)
      for (int i = 0; i < n; ++i) y[(long)i * N + k] = ycm[k * n + i];
  *st = c->st;
  free(mem); free(piv); free(ycm);
  return c->st.status;
}

void orc_integrate_batch(const orc_problem *proto, const orc_opts *o, double t0, double tf,
                         int64_t N, int64_t c0, int64_t c1, double *y, const double *fext,
                         const double *rho, orc_stats *st)
{
  int n = proto->n;
  for (int64_t c = c0; c < c1; ++c) {
    orc_problem p = *proto;
    double yc[ORC_NMAX], fc[ORC_NMAX];
    for (int k = 0; k < n; ++k) yc[k] = y[k * N + c];
    if (fext) {
      for (int k = 0; k < n; ++k) fc[k] = fext[k * N + c];
      p.fext = fc;
    } else {
      p.fext = NULL;
    }
    if (rho) p.rho = rho[c];
    orc_integrate(&p, o, t0, tf, yc, &st[c - c0], NULL);
    for (int k = 0; k < n; ++k) y[k * N + c] = yc[k];
  }
}
