/*
 * oracle.h -- CPU oracle for the batched BDF hot path (arXiv 2405.01713).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link,
 * load or execute anything under oracle/.  The only permitted users are
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs.  The oracle shares no code, header, table or
 * constant generator with the CUDA path (paper_2405_01713_b200/csrc).
 *
 * Plain, slow, obviously-correct fp64 C99, one cell at a time.  Compiled with
 * -O2 -ffp-contract=off so that a*b+c is never fused behind our back; fma()
 * is called only where the listing (LU_FACTOR / LU_SOLVE)
 * prescribes it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * "listing" = SURVEY.md §8(c).2, the step-by-step reconstruction of CVODE's
 * fixed-leading-coefficient Nordsieck BDF that the paper defers to
 * (hindmarsh2005sundials).  Readings R1..R24 are SURVEY.md §8(c).3 and
 * are restated in DESIGN.md.
 *
 * Parity pins: see tests/test_oracle_*.py.  Every function below is pinned by
 * at least one test against something other than itself (closed forms,
 * published values, brute force, invariants) -- except where the header of a
 * function says "parity unpinned".
 */
#ifndef BDFB_ORACLE_H
#define BDFB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_QMAX 5          /* listing §8c.1: QMAX */
#define ORC_NMAX 64         /* largest system the oracle handles (n <= 64) */
#define ORC_MAXL 64         /* largest GMRES Krylov dimension (the integrator uses maxl = 5) */

/* ---- models -------------------------------------------- */
enum {
  ORC_MODEL_LINEAR = 0,     /* y' = lambda .* y + f_ext  (closed-form pins) */
  ORC_MODEL_ROBERTSON = 1,  /* S:180, §8c.6 C1 */
  ORC_MODEL_KWH = 2,        /* Nyx-style heating/cooling, §8c.6 C2, Appendix B */
  ORC_MODEL_MECH = 3        /* constant-volume reactor, §8c.6 C3-C5 */
};

/* linear-solver choice inside Newton (P:399 dense direct, P:480 CVDiag) */
/* ORC_LS_DENSE_DQ: dense direct solver with the difference-quotient Jacobian (the paper's approaches 3A/3B,
 * P:177-178) instead of the analytic one (2A/2B) */
/* ORC_LS_GMRES: inexact Newton-Krylov, scaled GMRES with the difference-quotient Jv product (approaches 1A/1B,
 * Table 1, Eq. 5-6; krylov.c and lsolve_gmres in bdf.c) */
enum { ORC_LS_DENSE = 0, ORC_LS_DIAG = 1, ORC_LS_DENSE_DQ = 2, ORC_LS_GMRES = 3 };

/* time-integration method (orc_opts.method): CVODE BDF (default) or the explicit adaptive ERK of P:415-426
 * (erk.c) */
enum { ORC_METHOD_BDF = 0, ORC_METHOD_ERK4 = 1 };

/* Jacobian source for the dense solver */
enum { ORC_JAC_ANALYTIC = 0 /* model's exact J: closed form or complex step */ };

/* per-cell status */
enum {
  ORC_OK = 0,
  ORC_TOO_MUCH_WORK = 1,
  ORC_ERR_FAILURE = 2,
  ORC_CONV_FAILURE = 3,
  ORC_RHS_FAIL = 4,
  ORC_NONFINITE_INPUT = 5
};

/* KWH96-form heating/cooling parameters (Appendix B; reading R21) */
typedef struct {
  double z;               /* redshift */
  double X, Y;            /* H and He mass fractions */
  double gamma_ad;        /* adiabatic index */
  double gph[3];          /* photo-ionisation rates H0, He0, He+  [1/s] */
  double eph[3];          /* photo-heating rates   H0, He0, He+  [erg/s] */
} orc_kwh_params;

/* Flattened reaction mechanism (constant-volume reactor, §8c.6).
 * Units: CHEMKIN cgs (mol, cm^3, s), Ea in cal/mol, T in K.
 * Species k = 0..K-1 hold mass fractions Y_k; state index K is T.        */
typedef struct {
  int K;                 /* number of species                          */
  int nr;                /* number of reactions                        */
  const double *W;       /* [K] molecular weights g/mol                */
  const double *nasa;    /* [K][15]: Tmid, a_low[7], a_high[7]         */
  const int *reac;       /* [I][3] reactant species, -1 = empty slot   */
  const int *prod;       /* [I][3] product species,  -1 = empty slot   */
  const int *rev;        /* [I] 1 = reversible via Kc                  */
  const int *type;       /* [I] 0 elementary, 1 three-body, 2 Lindemann, 3 Troe */
  const double *arr;     /* [I][3] A, beta, Ea (k_inf for falloff)     */
  const double *arr0;    /* [I][3] A0, beta0, Ea0 (falloff low-p limit)*/
  const double *troe;    /* [I][4] a, T3, T1, T2 (T2 used iff has_t2)  */
  const int *has_t2;     /* [I]                                        */
  const double *eff;     /* [I][K] third-body efficiencies             */
} orc_mech;

typedef struct {
  int kind;              /* ORC_MODEL_* */
  int n;                 /* system size */
  const double *lambda;  /* LINEAR: [n] rates */
  const double *rob_k;   /* ROBERTSON: k1,k2,k3 */
  const orc_kwh_params *kwh;
  const orc_mech *mech;
  double rho;            /* per-cell aux: density g/cm^3 (KWH, MECH) */
  const double *fext;    /* per-cell frozen forcing F, [n] or NULL */
} orc_problem;

typedef struct {
  double rtol;
  const double *atol;    /* [n] */
  int qmax;              /* 1..5 */
  int64_t mxstep;        /* R12: per outer step */
  double h0;             /* 0 = cvHin */
  double hmin, hmax;     /* hmax <= 0 means infinity */
  int ls;                /* ORC_LS_DENSE | ORC_LS_DIAG | ORC_LS_DENSE_DQ */
  int group;             /* G: WRMS summation order emulation (R15); 1 = sequential */
  int method;            /* ORC_METHOD_BDF | ORC_METHOD_ERK4 (orc_integrate dispatches on it) */
  int maxl;              /* ORC_LS_GMRES: Krylov dimension cap (0 = 5, CVODE's default; reading R29) */
  int plain;             /* 1: the listing's plain arithmetic -- libm pow(x, 1.0/L) for the step-size
                            factors and true division in LU_SOLVE -- instead of readings R25/R16 (the
                            GPU's division-free root and reciprocal-multiply solve).  The GPU must match
                            both modes within the end-state band; it is bit-identical to plain = 0 only. */
} orc_opts;

typedef struct {
  int32_t status;
  int32_t nst, nfe, nje, nsetups, nni, netf, ncfn;
  int32_t q_last;
  double h_last;
  double t_reached;
  int32_t nli;           /* ORC_LS_GMRES: linear (Krylov) iterations; their Jv RHS calls are not in nfe */
} orc_stats;

/* optional trace of accepted steps, for the Nordsieck invariant pin */
typedef struct {
  int cap;               /* records available */
  int count;             /* records written */
  double *tn;            /* [cap] */
  double *h;             /* [cap] */
  int *q;                /* [cap] */
  double *zn;            /* [cap][ORC_QMAX+1][n] */
} orc_trace;

#define ORC_GBLK 256        /* global-norm mode: cells per partial sum (R15) */

/* ---- primitives -------------------------------------------------------- */
double orc_wrms(int n, const double *v, const double *w, int group);

/* Typical values and tolerances (Eq. 7).
 * orc_typical_values: y is YC (y[k*ncells + c]); tv[k] = 1/2 (min_c y[k][c] + max_c y[k][c])
 *   ("the min and max operations are taken over the entire computational domain"); min/max by
 *   C99 fmin/fmax (a NaN entry is skipped unless the whole component is NaN).  ncells >= 1.
 * orc_atol_from_typical: atol[k] = max(eta * tv[k], floor) (Eq. 7 with the SPEC's positive floor,
 *   the paper leaves tv = 0 undefined).                                             */
void orc_typical_values(int n, int64_t ncells, const double *y, double *tv);
void orc_atol_from_typical(int n, const double *tv, double eta, double floor_, double *atol);
double orc_wrms_sum(int n, const double *v, const double *w, int group);
int orc_lu_factor(int n, double *M /* row-major n*n, in/out */, int *piv);
void orc_lu_solve(int n, const double *LU, const int *piv, double *b);
/* the listing's LU_SOLVE with true division b[k] /= U[k][k] (plain mode) */
void orc_lu_solve_div(int n, const double *LU, const int *piv, double *b);

/* PREPARE_NEXT scalar part (cvChooseEta + cvSetEta) for the controller pins:
 * q, *qwait (in/out), etamax, h, hmax (<= 0: none), dsm = ||LTE||, ddn =
 * ||zn[q]|| tq[1] (q > 1), dup = ||acor - c zn[qmax]|| tq[3] (iff have_up),
 * plain: pow instead of R25.  Returns eta; sets *qprime, *hprime.          */
double orc_choose_eta(int q, int *qwait, double etamax, double h, double hmax, double dsm, double ddn,
                      int have_up, double dup, int plain, int *qprime, double *hprime);

/* One Newton solve of the listing (forced matrix setup with J at zn0) for
 * the Newton replay pin; see bdf.c.  Returns 0 / 1 (recoverable) / 2.      */
int orc_newton_once(const orc_problem *p, const orc_opts *o, double tn, double h, double rl1, double tol,
                    const double *zn0, const double *zn1, const double *ewt, double *acor, double *acnrm,
                    int *nni, int *nfe);

/* Scaled GMRES (krylov.c; Eq. 5-6).  Solves A x = b through A~ = S1 A S2^-1 with S1 = diag(s1),
 * S2 = diag(s2) (NULL = identity), zero initial guess, at most maxl (<= ORC_MAXL) iterations, no restarts;
 * converged when the rotation residual ||S1 (b - A x)||_2 <= delta.  atimes(ctx, v, z) sets z = A v and
 * returns 0, > 0 (recoverable failure) or < 0.  Outputs x, the iteration count and the final rotation
 * residual.  Returns ORC_GMRES_*: SUCCESS; RES_REDUCED (cap reached, residual below ||S1 b||: x is the best
 * iterate); CONV_FAIL; ATIMES_FAIL_REC / _UNREC; QRFACT_FAIL / QRSOL_FAIL (zero diagonal in the rotated
 * Hessenberg matrix).                                                                                    */
typedef int (*orc_atimes_fn)(void *ctx, const double *v, double *z);
enum { ORC_GMRES_SUCCESS = 0, ORC_GMRES_RES_REDUCED = 1, ORC_GMRES_CONV_FAIL = 2, ORC_GMRES_ATIMES_FAIL_REC = 3,
       ORC_GMRES_QRFACT_FAIL = 4, ORC_GMRES_QRSOL_FAIL = 5, ORC_GMRES_ATIMES_FAIL_UNREC = -1 };
int orc_gmres(int n, int maxl, orc_atimes_fn atimes, void *ctx, const double *b, const double *s1,
              const double *s2, double delta, double *x, int *nli, double *res_norm);

/* Explicit adaptive ERK (erk.c): one step of the embedded 4(3) pair from (t, y)
 * with step h: ynew (order 4) and err = h sum_i e_i k_i (the order-4 minus order-3 difference, the LTE
 * estimate).  Returns 0 or the RHS status of the first failing stage.  nfe: RHS calls made (5, or 4 when
 * k1 != NULL supplies f(t, y)).                                                                           */
int orc_erk_step(const orc_problem *p, double t, double h, const double *y, const double *k1, double *ynew,
                 double *err, int *nfe);

/* f = R(t,y) + f_ext.  Returns 0, or >0 for a recoverable RHS failure. */
int orc_rhs(const orc_problem *p, double t, const double *y, double *f);
/* S_i: the RHS with |.| on every term (reading R19 parity scale). */
int orc_rhs_scale(const orc_problem *p, double t, const double *y, double *S);
/* J = d f / d y (row-major).  Analytic (LINEAR, ROBERTSON) or complex-step
 * (MECH).  Returns 0 or >0 on failure.  KWH has no J (CVDiag only).       */
int orc_jac(const orc_problem *p, double t, const double *y, double *J);
/* Difference-quotient dense Jacobian (CVODE's cvLsDenseDQJac, the reading of the paper's "finite
 * difference" Jacobian): srur = sqrt(u), fnorm = ||fy||_WRMS(ewt) (sequential order),
 * minInc = 1000 |h| u n fnorm (1 if fnorm = 0); column j: inc = max(srur |y_j|, minInc / ewt_j),
 * J(:, j) = (1/inc) f(t, y + inc e_j) + (-(1/inc)) fy.  fy = f(t, y).  Returns 0 or the RHS failure. */
int orc_jac_dq(const orc_problem *p, double t, const double *y, const double *fy, const double *ewt, double h,
               double *J);

/* KWH pin entry: converged ionisation state for energy e:
 * out8 = [T, n_H0, n_H+, n_He0, n_He+, n_He++, n_e, g(x_e)]              */
int orc_kwh_state(const orc_problem *p, double e, double *out8);

/* x^(1/L) by the fixed IEEE sequence of reading R25 (step-size factors) */
double orc_root(double x, int L);

/* cvSetBDF + cvSetTqBDF for the coefficient pins: l[0..5], tq[1..5] */
void orc_set_bdf(int q, double h, const double *tau /* [7], tau[1..6] */,
                 int qwait, double *l, double *tq);

/* Integrate one cell from t0 to tf in place (y: [n]).  Returns status.
 * o->method == ORC_METHOD_ERK4 integrates with the explicit ERK (orc_integrate_erk).                     */
int orc_integrate(const orc_problem *p, const orc_opts *o, double t0,
                  double tf, double *y, orc_stats *st, orc_trace *tr);

/* The explicit adaptive ERK integration of one cell (erk.c; WRMS error control of Eq. 3 with the
 * embedded estimate, reading R30).  Uses o->rtol, atol, mxstep, h0, hmin, hmax.  Returns status.         */
int orc_integrate_erk(const orc_problem *p, const orc_opts *o, double t0, double tf, double *y, orc_stats *st);

/* Global-norm mode: the N cells of a YC field integrated as one system with
 * batch-wide norms (see bdf.c).  fext YC or NULL, rho [N] or NULL.          */
int orc_integrate_global(const orc_problem *proto, const orc_opts *o, double t0, double tf,
                         int64_t N, double *y, const double *fext, const double *rho,
                         orc_stats *st);

/* Batch driver over cells [c0, c1) of a YC (component-major) field:
 * y[k*N + c], fext[k*N + c] (or NULL), rho[c] (or NULL).  Stats written
 * per cell into st[c - c0].  Model parameters come from *proto (its rho and
 * fext fields are overwritten per cell).                                  */
void orc_integrate_batch(const orc_problem *proto, const orc_opts *o,
                         double t0, double tf, int64_t N, int64_t c0,
                         int64_t c1, double *y, const double *fext,
                         const double *rho, orc_stats *st);

#ifdef __cplusplus
}
#endif
#endif
