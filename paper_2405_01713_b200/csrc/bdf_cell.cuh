// bdf_cell.cuh -- the per-cell BDF integrator as a persistent, resumable
// state machine (B200 / sm_100a).
//
// Semantics: CVODE's fixed-leading-coefficient Nordsieck BDF, orders 1..5,
// exactly as the step-by-step listing SURVEY.md §8(c).2 (the algorithm the
// paper defers to): INIT/HIN,
// O1-O5 outer loop, STEP (PREDICT, SET_BDF, NEWTON, error test, RESTORE,
// RESCALE, ADJUST_ORDER), DONE, PREPARE_NEXT, SET_ETA.  Constants: listing
// §8(c).1.  This is an independent implementation (no code shared with
// oracle/), organised for the GPU:
//
//  * one cell per group of G lanes (grp.cuh); all scalar state replicated in
//    the group's registers; vectors distributed one component per lane (or
//    all components in one thread for G = 1);
//  * Nordsieck history zn[0..5], weights, corrections in REGISTERS; saved J
//    and the LU factors in shared memory (lu.cuh);
//  * a flat state machine whose only convergence point is the model RHS:
//    every trip around the loop advances each group's cell to its next RHS
//    request (predictor, Newton residual, CVDiag perturbation, cvHin probe,
//    error-test restart, or a fresh cell), then all groups evaluate the RHS
//    together.  Lanes of different groups may be at different steps of
//    different cells (per-cell adaptive stepping with masked lanes: a stiff
//    cell never stalls an easy one);
//  * a persistent grid that pulls cells (chunks of CHUNK consecutive cells)
//    from a device work counter, so per-cell cost variance is load-balanced;
//  * no host round trips, no allocation, one launch per integrate.
#pragma once
#include <float.h>
#include <stdint.h>
#include "grp.cuh"
#include "lu.cuh"

namespace bdfb {

// ---- listing §8c.1 constants --------------------------------------------------
constexpr int QMAX = 5;
constexpr double NLSCOEF = 0.1, CRDOWN = 0.3, RDIV = 2.0, DGMAX = 0.3, DGMAX_JBAD = 0.2;
constexpr int MAXCOR = 3, MSBP = 20, MSBJ = 51;
constexpr double BIAS1 = 6.0, BIAS2 = 6.0, BIAS3 = 10.0, ADDON = 1e-6, THRESH = 1.5;
constexpr double ETAMX1 = 1e4, ETAMX2 = 10.0, ETAMIN = 0.1, ETAMXF = 0.2, ETACF = 0.25;
constexpr int SMALL_NEF = 2, MXNEF1 = 3, MXNEF = 7, MXNCF = 10, LONG_WAIT = 10, HIN_ITERS = 4;
constexpr double HUB_FACTOR = 0.1, H_BIAS = 0.5, FRACT = 0.1;
constexpr double UROUND = DBL_EPSILON;

enum : int { ST_OK = 0, ST_TOO_MUCH_WORK = 1, ST_ERR_FAILURE = 2, ST_CONV_FAILURE = 3, ST_RHS_FAIL = 4,
             ST_NONFINITE = 5 };
enum : int { NF_FIRST = 0, NF_PREV_CONV = 1, NF_PREV_ERR = 2 };
enum : int { CF_NONE = 0, CF_BAD_J = 1, CF_OTHER = 2 };
// RHS-request phases (what to do with the next RHS value)
enum : int { PH_INIT = 0, PH_HIN = 1, PH_NRES = 2, PH_DIAG = 3, PH_ETF3 = 4, PH_DONE = 5 };

struct Opts {
  double rtol;
  double t0, tf;
  double h0, hmin, hmax;      // hmax <= 0: unlimited
  long long mxstep;
  int qmax;
  int layout;                 // 0 YC, 1 CY
  long long ncells;
};

struct CellStatsPtrs {
  int *status, *nst, *nfe, *nje, *nsetups, *nni, *netf, *ncfn, *q_last;
  double *h_last, *t_reached;
};

struct Agg {  // device aggregate counters (unsigned long long for atomics)
  unsigned long long n_failed, nst, nfe, nje, nsetups, nni, netf, ncfn, nst_max, nfe_max, cells_done;
  unsigned long long nli;   // GMRES linear iterations (SPLIT LS_GMRES only)
};

template <int N, int R>
struct Vec {
  double v[R];
};

// x^(1/L) for the step-size factors, reading R25: instead of
// pow(x, 1.0/L) the real L-th root by a fixed, division-free IEEE operation
// sequence, so that CPU and GPU step-size decisions are bit-reproducible:
//   x = y 2^e (y in [1,2)), e = L k + r;  s ~ y^(-1/L) from s0 = 1-(y-1)c_L
//   and 4 Newton steps s <- s (1 + (1 - y s^L)/L);  x^(1/L) = ldexp(y s^(L-1)
//   2^(r/L), k).  c_L = 1 - 2^(-1/L) and 2^(r/L): correctly rounded constants.
// Compiled with -fmad=false: no contraction changes the sequence.
__constant__ double kRootC[8][7] = {
    {0}, {1.0},
    {0x1.0p+0, 0x1.6a09e667f3bcdp+0},
    {0x1.0p+0, 0x1.428a2f98d728bp+0, 0x1.965fea53d6e3dp+0},
    {0x1.0p+0, 0x1.306fe0a31b715p+0, 0x1.6a09e667f3bcdp+0, 0x1.ae89f995ad3adp+0},
    {0x1.0p+0, 0x1.2611186bae675p+0, 0x1.51cb453b9536cp+0, 0x1.8406003b2ae5cp+0, 0x1.bdb8cdadbe120p+0},
    {0x1.0p+0, 0x1.1f59ac3c7d6c0p+0, 0x1.428a2f98d728bp+0, 0x1.6a09e667f3bcdp+0, 0x1.965fea53d6e3dp+0,
     0x1.c823e074ec129p+0},
    {0x1.0p+0, 0x1.1aa59c4115e7dp+0, 0x1.381147622f886p+0, 0x1.588cea3f093bep+0, 0x1.7c6a1f29e2ce6p+0,
     0x1.a402feeb9c533p+0, 0x1.cfbb031a741a5p+0}};
__constant__ double kRootCL[8] = {0, 0, 0x1.2bec333018867p-2, 0x1.a68056b0a470ep-3, 0x1.45d819a94b14bp-3,
                                  0x1.091cc94907b7fp-3, 0x1.bee0fc589f6b6p-4, 0x1.8227e72c5f2dbp-4};
__constant__ double kInvL[8] = {0, 1.0 / 1, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7};

static __device__ __noinline__ double root_l(double x, int L) {
  if (!(x > 0.0) || isinf(x)) return x > 0.0 ? x : 0.0;
  if (L == 1) return x;
  int e;
  const double y = 2.0 * frexp(x, &e);
  e = e - 1;
  const int k = (e >= 0) ? e / L : -((-e + L - 1) / L);
  const int r = e - L * k;
  const double invL = kInvL[L];
  double s = 1.0 - (y - 1.0) * kRootCL[L];
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    double p = s;
#pragma unroll
    for (int j = 0; j < 6; ++j)
      if (j < L - 1) p = p * s;
    s = s * (1.0 + (1.0 - y * p) * invL);
  }
  double t = y;
#pragma unroll
  for (int j = 0; j < 6; ++j)
    if (j < L - 1) t = t * s;
  return ldexp(t * kRootC[L][r], k);
}

// select arr[idx] for a small register array without dynamic indexing
template <int M>
__device__ __forceinline__ double sel(const double (&a)[M], int idx) {
  double r = a[0];
#pragma unroll
  for (int i = 1; i < M; ++i)
    if (i == idx) r = a[i];
  return r;
}

template <class Model>
struct Integrator {
  static constexpr int N = Model::N;
  static constexpr int G = Model::G;
  static constexpr int R = (N + G - 1) / G;
  static constexpr bool DIAG = Model::DIAG;
  static constexpr int CHUNK = (G == 1) ? 1 : 4;
  static constexpr int MAT = (G == 1 ? N * N : N) * WS;          // doubles per matrix per warp
  // the LU area also hosts the Jacobian's scratch (the setup overwrites it)
  static constexpr int MATLU = MAT > Model::JSCRATCH ? MAT : Model::JSCRATCH;
  static constexpr int SMEM_WARP = (DIAG ? 0 : MAT + MATLU) + Model::SCRATCH + 16;  // + perm ints (32)
  using Lay = Layout<N, G>;
  using P = typename Model::Params;

  // ------------------------------------------------------------------ state
  struct S {
    double zn[QMAX + 1][R];
    double ewt[R], acor[R], fy[R], yq[R], del[R], atol[R], fext[R], minv[R];
    double aux;
    double tn, tq_req, h, hscale, hprime, eta, etamax, saved_t;
    double tau[QMAX + 2], l[QMAX + 1], tq[6];
    double rl1, gamma, gammap, gamrat, crate, acnrm, saved_tq5, dprev, gammasv, tol;
    double hg, hs, hub, hnew;   // cvHin
    int q, qprime, L, qwait;
    int nst, nfe, nje, nsetups, nni, netf, ncfn;
    int nstlp, nstlj, nef, ncf, nflag, convfail, setup, jcur, m;
    int count1, count2;
    int phase, status;
    long long cell, chunk_end;
    int pos;             // G > 1 LU position
    double invd;         // G > 1: 1 / U diagonal of this lane's row
    int piv[N];          // G = 1 LU pivots (static indexing only)
  };

  // ---------------------------------------------------------------- helpers
  __device__ static double wrms(const Grp<G>& g, const double (&v)[R], const double (&w)[R]) {
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (Lay::valid(g.lane, r)) {
        double p = v[r] * w[r];
        acc = acc + p * p;
      }
    return sqrt(g.sum(acc) / (double)N);
  }

  __device__ static void set_ewt(const Opts& o, S& s, const double (&y)[R]) {
#pragma unroll
    for (int r = 0; r < R; ++r) s.ewt[r] = 1.0 / (o.rtol * fabs(y[r]) + s.atol[r]);
  }

  __device__ static void rescale(S& s) {
    double f = s.eta;
#pragma unroll
    for (int j = 1; j <= QMAX; ++j) {
      if (j <= s.q) {
#pragma unroll
        for (int r = 0; r < R; ++r) s.zn[j][r] = f * s.zn[j][r];
        f = f * s.eta;
      }
    }
    s.h = s.hscale * s.eta;
    s.hscale = s.h;
  }

  __device__ static void predict(const Opts& o, S& s) {
    s.tn = s.tn + s.h;
    if ((s.tn - o.tf) * s.h > 0.0) s.tn = o.tf;
#pragma unroll
    for (int k = 1; k <= QMAX; ++k)
#pragma unroll
      for (int j = QMAX; j >= 1; --j)
        if (k <= s.q && j >= k && j <= s.q) {
#pragma unroll
          for (int r = 0; r < R; ++r) s.zn[j - 1][r] = s.zn[j - 1][r] + s.zn[j][r];
        }
  }

  __device__ static void restore(S& s) {
    s.tn = s.saved_t;
#pragma unroll
    for (int k = 1; k <= QMAX; ++k)
#pragma unroll
      for (int j = QMAX; j >= 1; --j)
        if (k <= s.q && j >= k && j <= s.q) {
#pragma unroll
          for (int r = 0; r < R; ++r) s.zn[j - 1][r] = s.zn[j - 1][r] - s.zn[j][r];
        }
  }

  // cvSetBDF + cvSetTqBDF, predicated so that only static register indices occur
  __device__ static void set_bdf(S& s) {
    const int q = s.q;
    const double h = s.h;
    double xi_inv = 1.0, xistar_inv = 1.0, alpha0 = -1.0, alpha0_hat = -1.0, hsum = h;
    s.l[0] = 1.0;
    s.l[1] = 1.0;
#pragma unroll
    for (int i = 2; i <= QMAX; ++i) s.l[i] = 0.0;
    if (q > 1) {
#pragma unroll
      for (int j = 2; j < QMAX; ++j) {
        if (j < q) {
          hsum = hsum + s.tau[j - 1];
          xi_inv = h / hsum;
          alpha0 = alpha0 - 1.0 / j;
#pragma unroll
          for (int i = QMAX; i >= 1; --i)
            if (i <= j) s.l[i] = s.l[i] + s.l[i - 1] * xi_inv;
        }
      }
      alpha0 = alpha0 - 1.0 / q;
      xistar_inv = -s.l[1] - alpha0;
      hsum = hsum + sel(s.tau, q - 1);
      xi_inv = h / hsum;
      alpha0_hat = -s.l[1] - xi_inv;
#pragma unroll
      for (int i = QMAX; i >= 1; --i)
        if (i <= q) s.l[i] = s.l[i] + s.l[i - 1] * xistar_inv;
    }
    const double lq = sel(s.l, q);
    const double A1 = 1.0 - alpha0_hat + alpha0;
    const double A2 = 1.0 + q * A1;
    s.tq[2] = fabs(A1 / (alpha0 * A2));
    s.tq[5] = fabs(A2 * xistar_inv / (lq * xi_inv));
    if (s.qwait == 1) {
      if (q > 1) {
        const double C = xistar_inv / lq;
        const double A3 = alpha0 + 1.0 / q;
        const double A4 = alpha0_hat + xi_inv;
        const double Cpinv = (1.0 - A4 + A3) / A3;
        s.tq[1] = fabs(C * Cpinv);
      } else {
        s.tq[1] = 1.0;
      }
      hsum = hsum + sel(s.tau, q);
      xi_inv = h / hsum;
      const double A5 = alpha0 - 1.0 / (q + 1);
      const double A6 = alpha0_hat - xi_inv;
      const double Cppinv = (1.0 - A6 + A5) / A2;
      s.tq[3] = fabs(Cppinv / (xi_inv * (q + 2) * A5));
    }
    s.tq[4] = NLSCOEF / s.tq[2];
  }

  // zn[j] for dynamic j (read) -- vector select
  __device__ static void zn_get(const S& s, int j, double (&out)[R]) {
#pragma unroll
    for (int r = 0; r < R; ++r) out[r] = s.zn[0][r];
#pragma unroll
    for (int jj = 1; jj <= QMAX; ++jj)
      if (jj == j) {
#pragma unroll
        for (int r = 0; r < R; ++r) out[r] = s.zn[jj][r];
      }
  }
  __device__ static void zn_set(S& s, int j, const double (&v)[R]) {
#pragma unroll
    for (int jj = 0; jj <= QMAX; ++jj)
      if (jj == j) {
#pragma unroll
        for (int r = 0; r < R; ++r) s.zn[jj][r] = v[r];
      }
  }

  __device__ static void increase_bdf(const Opts& o, S& s) {
    double l[QMAX + 1];
#pragma unroll
    for (int i = 0; i <= QMAX; ++i) l[i] = 0.0;
    double alpha1 = 1.0, prod = 1.0, xiold = 1.0, alpha0 = -1.0, hsum = s.hscale;
    l[2] = 1.0;
    if (s.q > 1) {
#pragma unroll
      for (int j = 1; j < QMAX; ++j) {
        if (j < s.q) {
          hsum = hsum + s.tau[j + 1];
          const double xi = hsum / s.hscale;
          prod = prod * xi;
          alpha0 = alpha0 - 1.0 / (j + 1);
          alpha1 = alpha1 + 1.0 / xi;
#pragma unroll
          for (int i = QMAX; i >= 2; --i)
            if (i <= j + 2) l[i] = l[i] * xiold + l[i - 1];
          xiold = xi;
        }
      }
    }
    const double A1 = (-alpha0 - alpha1) / prod;
    double zq[R], zL[R];
    zn_get(s, o.qmax, zq);
#pragma unroll
    for (int r = 0; r < R; ++r) zL[r] = A1 * zq[r];
    zn_set(s, s.q + 1, zL);
#pragma unroll
    for (int j = 2; j <= QMAX; ++j)
      if (j <= s.q) {
#pragma unroll
        for (int r = 0; r < R; ++r) s.zn[j][r] = l[j] * zL[r] + s.zn[j][r];
      }
  }

  __device__ static void decrease_bdf(S& s) {
    double l[QMAX + 1];
#pragma unroll
    for (int i = 0; i <= QMAX; ++i) l[i] = 0.0;
    l[2] = 1.0;
    double hsum = 0.0;
#pragma unroll
    for (int j = 1; j <= QMAX - 2; ++j) {
      if (j <= s.q - 2) {
        hsum = hsum + s.tau[j];
        const double xi = hsum / s.hscale;
#pragma unroll
        for (int i = QMAX; i >= 2; --i)
          if (i <= j + 2) l[i] = l[i] * xi + l[i - 1];
      }
    }
    double zq[R];
    zn_get(s, s.q, zq);
#pragma unroll
    for (int j = 2; j < QMAX; ++j)
      if (j < s.q) {
#pragma unroll
        for (int r = 0; r < R; ++r) s.zn[j][r] = -l[j] * zq[r] + s.zn[j][r];
      }
  }

  __device__ static void adjust_order(const Opts& o, S& s, int dq) {
    if (s.q == 2 && dq != 1) return;
    if (dq == 1) increase_bdf(o, s);
    else decrease_bdf(s);
  }

  __device__ static void set_eta(const Opts& o, S& s) {
    if (s.eta < THRESH) {
      s.eta = 1.0;
      s.hprime = s.h;
    } else {
      s.eta = fmin(s.eta, s.etamax);
      if (o.hmax > 0.0) s.eta = s.eta / fmax(1.0, fabs(s.h) * s.eta / o.hmax);
      s.hprime = s.h * s.eta;
    }
  }

  __device__ static void prepare_next(const Grp<G>& g, const Opts& o, S& s, double dsm) {
    if (s.etamax == 1.0) {
      s.qwait = s.qwait > 2 ? s.qwait : 2;
      s.qprime = s.q;
      s.hprime = s.h;
      s.eta = 1.0;
      return;
    }
    const double etaq = 1.0 / (root_l(BIAS2 * dsm, s.L) + ADDON);
    if (s.qwait != 0) {
      s.eta = etaq;
      s.qprime = s.q;
      set_eta(o, s);
      return;
    }
    s.qwait = 2;
    double etaqm1 = 0.0, etaqp1 = 0.0;
    if (s.q > 1) {
      double zq[R];
      zn_get(s, s.q, zq);
      const double ddn = wrms(g, zq, s.ewt) * s.tq[1];
      etaqm1 = 1.0 / (root_l(BIAS1 * ddn, s.q) + ADDON);
    }
    if (s.q != o.qmax && s.saved_tq5 != 0.0) {
      const double hr = s.h / s.tau[2];
      double pw = 1.0;
#pragma unroll
      for (int k = 0; k < QMAX + 1; ++k)
        if (k < s.L) pw = pw * hr;
      const double cquot = (s.tq[5] / s.saved_tq5) * pw;
      double zq[R], t[R];
      zn_get(s, o.qmax, zq);
#pragma unroll
      for (int r = 0; r < R; ++r) t[r] = -cquot * zq[r] + s.acor[r];
      const double dup = wrms(g, t, s.ewt) * s.tq[3];
      etaqp1 = 1.0 / (root_l(BIAS3 * dup, s.L + 1) + ADDON);
    }
    const double etam = fmax(etaqm1, fmax(etaq, etaqp1));
    if (etam < THRESH) {
      s.eta = 1.0;
      s.qprime = s.q;
    } else if (etam == etaq) {
      s.eta = etaq;
      s.qprime = s.q;
    } else if (etam == etaqm1) {
      s.eta = etaqm1;
      s.qprime = s.q - 1;
    } else {
      s.eta = etaqp1;
      s.qprime = s.q + 1;
      zn_set(s, o.qmax, s.acor);
    }
    set_eta(o, s);
  }

  // ------------------------------------------------------------- linear algebra
  // dense setup: optional J evaluation (into Jm), M = I - gamma J into LUm, factor
  __device__ static int lsetup_dense(const Grp<G>& g, const P& prm, S& s, double* Jm, double* LUm, int* perm,
                                     double* scratch) {
    int rv = 0;
    const double dgamma = fabs(s.gamma / s.gammap - 1.0);
    const bool jbad = (s.nst == 0) || (s.nst >= s.nstlj + MSBJ) ||
                      (s.convfail == CF_BAD_J && dgamma < DGMAX_JBAD) || (s.convfail == CF_OTHER);
    if (jbad) {
      s.nje++;
      s.nstlj = s.nst;
      s.jcur = 1;
      if (Model::jac(g, prm, s.tn, s.yq, s.aux, Jm, scratch, LUm)) rv = -1;
    } else {
      s.jcur = 0;
    }
    if (rv == 0) {
      if constexpr (G == 1) {
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int j = 0; j < N; ++j)
            mat<N, G>(LUm, g, i, j) = (i == j ? 1.0 : 0.0) - s.gamma * mat<N, G>(Jm, g, i, j);
        rv = lu_factor_thread<N>(g, LUm, s.piv) ? 1 : 0;
      } else {
        if (g.lane < N) {
#pragma unroll 4
          for (int j = 0; j < N; ++j)
            LUm[j * WS + g.wlane] = (g.lane == j ? 1.0 : 0.0) - s.gamma * Jm[j * WS + g.wlane];
        }
        g.sync();
        rv = lu_factor_group<N, G>(g, LUm, s.pos, perm) ? 1 : 0;
        if (!rv) s.invd = lu_inv_diag<N, G>(g, LUm, s.pos);
      }
    }
    s.nsetups++;
    s.gamrat = 1.0;
    s.gammap = s.gamma;
    s.crate = 1.0;
    s.nstlp = s.nst;
    return rv;
  }

  // b <- M^{-1} b
  __device__ static int lsolve(const Grp<G>& g, S& s, const double* LUm, const int* perm, double (&b)[R]) {
    if constexpr (DIAG) {
      if (s.gammasv != s.gamma) {
        const double rr = s.gamma / s.gammasv;
        int bad = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double Mi = (1.0 / s.minv[r] + (-1.0)) * rr + 1.0;
          if (Lay::valid(g.lane, r) && Mi == 0.0) bad = 1;
          s.minv[r] = 1.0 / Mi;
        }
        if (g.ior(bad)) return 1;
        s.gammasv = s.gamma;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) b[r] = b[r] * s.minv[r];
      return 0;
    } else {
    if constexpr (G == 1) {
      double bb[N];
#pragma unroll
      for (int i = 0; i < N; ++i) bb[i] = b[i];
      lu_solve_thread<N>(g, LUm, s.piv, bb);
#pragma unroll
      for (int i = 0; i < N; ++i) b[i] = bb[i];
    } else {
      b[0] = lu_solve_group<N, G>(g, LUm, s.pos, s.invd, perm, b[0]);
    }
    if (s.gamrat != 1.0) {
      const double sc = 2.0 / (1.0 + s.gamrat);
#pragma unroll
      for (int r = 0; r < R; ++r) b[r] = sc * b[r];
    }
    return 0;
    }
  }

  // ------------------------------------------------------------------- I/O
  __device__ static long long idx(const Opts& o, long long c, int k) {
    return o.layout == 0 ? (long long)k * o.ncells + c : c * (long long)N + k;
  }

  // ---------------------------------------------------------------- kernel
  // Advance the state machine of this group's cell to its next RHS request.
  // Returns false when the group has no more cells.
  __device__ static bool advance(const Grp<G>& g, const Opts& o, const P& prm, S& s, int rv, double (&fr)[R],
                                 double* y, const double* fext, const double* aux, double* Jm, double* LUm,
                                 int* perm, double* scratch, unsigned long long* counter, Agg& acc,
                                 const CellStatsPtrs& cs) {
    enum { A_LOAD, A_STEP_TOP, A_ATTEMPT, A_SOLVE, A_NFAIL, A_ERRTEST, A_STORE, A_START, A_HIN_FINISH,
           A_REQ_RES };
    int act;
    switch (s.phase) {
      case PH_INIT: act = -1; break;
      case PH_HIN: act = -2; break;
      case PH_NRES: act = -3; break;
      case PH_DIAG: act = -4; break;
      case PH_ETF3: act = -5; break;
      default: act = A_LOAD; break;
    }
    double dsm = 0.0;
    for (;;) {
      switch (act) {
        // ------------------------------------------------------ RHS consumers
        case -1: {  // f(t0, y0) ready
          if (rv) { s.status = ST_RHS_FAIL; act = A_STORE; break; }
#pragma unroll
          for (int r = 0; r < R; ++r) s.zn[1][r] = fr[r];
          if (o.h0 != 0.0) { s.hnew = o.h0; act = A_START; s.h = o.h0; break; }
          // cvHin preamble (cvUpperBoundH0)
          const double tdist = o.tf - o.t0;
          const double tround = UROUND * fmax(fabs(o.t0), fabs(o.tf));
          const double hlb = 100.0 * tround;
          double hi = 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (Lay::valid(g.lane, r)) {
              const double d = HUB_FACTOR * fabs(s.zn[0][r]) + 1.0 / s.ewt[r];
              hi = fmax(hi, fabs(s.zn[1][r]) / d);
            }
          const double hub_inv = g.max(hi);
          double hub = HUB_FACTOR * tdist;
          if (hub * hub_inv > 1.0) hub = 1.0 / hub_inv;
          s.hub = hub;
          s.hg = sqrt(hlb * hub);
          if (hub < hlb) { s.h = s.hg; act = A_START; break; }
          s.hs = s.hg;
          s.hnew = s.hg;
          s.count1 = 1;
          s.count2 = 1;
#pragma unroll
          for (int r = 0; r < R; ++r) s.yq[r] = s.hg * s.zn[1][r] + s.zn[0][r];
          s.tq_req = o.t0 + s.hg;
          s.phase = PH_HIN;
          return true;
        }
        case -2: {  // cvYddNorm probe ready
          if (rv) {
            s.hg = s.hg * 0.2;
            s.count2++;
            if (s.count2 > HIN_ITERS) {
              if (s.count1 <= 2) { s.status = ST_RHS_FAIL; act = A_STORE; break; }
              s.hnew = s.hs;
              act = A_HIN_FINISH;
              break;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) s.yq[r] = s.hg * s.zn[1][r] + s.zn[0][r];
            s.tq_req = o.t0 + s.hg;
            return true;
          }
          const double ih = 1.0 / s.hg;
          double t[R];
#pragma unroll
          for (int r = 0; r < R; ++r) t[r] = (fr[r] - s.zn[1][r]) * ih;
          const double ydd = wrms(g, t, s.ewt);
          s.hs = s.hg;
          s.hnew = (ydd * s.hub * s.hub > 2.0) ? sqrt(2.0 / ydd) : sqrt(s.hg * s.hub);
          if (s.count1 == HIN_ITERS) { act = A_HIN_FINISH; break; }
          const double hrat = s.hnew / s.hg;
          if (hrat > 0.5 && hrat < 2.0) { act = A_HIN_FINISH; break; }
          if (s.count1 > 1 && hrat > 2.0) { s.hnew = s.hg; act = A_HIN_FINISH; break; }
          s.hg = s.hnew;
          s.count1++;
          s.count2 = 1;
#pragma unroll
          for (int r = 0; r < R; ++r) s.yq[r] = s.hg * s.zn[1][r] + s.zn[0][r];
          s.tq_req = o.t0 + s.hg;
          return true;
        }
        case A_HIN_FINISH: {
          const double tround = UROUND * fmax(fabs(o.t0), fabs(o.tf));
          const double hlb = 100.0 * tround;
          double h = H_BIAS * s.hnew;
          if (h < hlb) h = hlb;
          if (h > s.hub) h = s.hub;
          s.h = h;
          act = A_START;
          break;
        }
        case A_START: {
          double h0 = s.h;
          if (h0 > o.tf - o.t0) h0 = o.tf - o.t0;
          if (o.hmax > 0.0 && h0 > o.hmax) h0 = o.hmax;
#pragma unroll
          for (int r = 0; r < R; ++r) s.zn[1][r] = h0 * s.zn[1][r];
          s.h = s.hscale = s.hprime = h0;
          s.q = s.qprime = 1;
          s.L = 2;
          s.qwait = 2;
          s.etamax = ETAMX1;
          s.crate = 1.0;
          s.eta = 1.0;
          act = A_STEP_TOP;
          break;
        }
        case -3: {  // Newton residual f(tn, zn0 + ycor) ready
          if (rv) {
            if (s.m == 0) s.jcur = 1;   // a failed first residual is not retried (reading R5)
            act = A_NFAIL;
            break;
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            s.fy[r] = fr[r];
            const double t = s.rl1 * s.zn[1][r] + s.acor[r];
            s.del[r] = -s.gamma * s.fy[r] + t;
          }
          if (s.setup) {
            if constexpr (DIAG) {
              const double rr = FRACT * s.rl1;
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const double ft = s.h * s.fy[r] - s.zn[1][r];
                s.yq[r] = rr * ft + s.yq[r];
              }
              s.phase = PH_DIAG;
              return true;
            } else {
              rv = lsetup_dense(g, prm, s, Jm, LUm, perm, scratch);
              s.setup = 0;
              if (rv) { rv = rv < 0 ? 1 : rv; act = A_NFAIL; break; }
            }
          }
          act = A_SOLVE;
          break;
        }
        case -4: {  // CVDiag perturbed RHS ready
          s.nje++;
          s.jcur = 1;
          int bad = rv ? 1 : 0;
          if (!rv) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const double ft = s.h * s.fy[r] - s.zn[1][r];
              double Mi;
              if (fabs(ft * s.ewt[r]) >= UROUND)
                Mi = (FRACT * ft + (-s.h) * (fr[r] - s.fy[r])) / (FRACT * ft);
              else
                Mi = 1.0;
              if (Lay::valid(g.lane, r) && Mi == 0.0) bad = 1;
              s.minv[r] = 1.0 / Mi;
            }
            s.gammasv = s.gamma;
          }
          bad = g.ior(bad);
          s.nsetups++;
          s.gamrat = 1.0;
          s.gammap = s.gamma;
          s.crate = 1.0;
          s.nstlp = s.nst;
          s.setup = 0;
          rv = bad;
          act = rv ? A_NFAIL : A_SOLVE;
          break;
        }
        case -5: {  // RHS at (tn, zn0) after the 3rd+ error-test failure at q = 1
          if (rv) { s.status = ST_RHS_FAIL; act = A_STORE; break; }
#pragma unroll
          for (int r = 0; r < R; ++r) s.zn[1][r] = s.h * fr[r];
          act = A_ATTEMPT;
          break;
        }

        // ------------------------------------------------------ new cell
        case A_LOAD: {
          if (s.cell + 1 < s.chunk_end) {
            s.cell++;
          } else {
            long long c0 = 0;
            if (g.lane == 0) c0 = (long long)atomicAdd(counter, (unsigned long long)CHUNK);
            c0 = __shfl_sync(g.mask, c0, 0, G);
            if (c0 >= o.ncells) { s.phase = PH_DONE; return false; }
            s.cell = c0;
            s.chunk_end = c0 + CHUNK < o.ncells ? c0 + CHUNK : o.ncells;
          }
          const long long c = s.cell;
          s.aux = aux ? aux[c] : 0.0;
          int bad = 0;
          double y0[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int k = Lay::comp(g.lane, r);
            if (k < N) {
              y0[r] = y[idx(o, c, k)];
              s.fext[r] = fext ? fext[idx(o, c, k)] : 0.0;
              if (!isfinite(y0[r]) || !isfinite(s.fext[r])) bad = 1;
            } else {
              y0[r] = 0.0;
              s.fext[r] = 0.0;
            }
          }
          if (!isfinite(s.aux)) bad = 1;
          bad = g.ior(bad);
          s.nst = s.nfe = s.nje = s.nsetups = s.nni = s.netf = s.ncfn = 0;
          s.nstlp = s.nstlj = 0;
          s.status = ST_OK;
          s.tn = o.t0;
          s.q = 1;
          s.h = 0.0;
#pragma unroll
          for (int j = 0; j <= QMAX; ++j)
#pragma unroll
            for (int r = 0; r < R; ++r) s.zn[j][r] = 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            s.zn[0][r] = y0[r];
            s.acor[r] = 0.0;
            s.minv[r] = 1.0;
          }
#pragma unroll
          for (int i = 0; i <= QMAX + 1; ++i) s.tau[i] = 0.0;
#pragma unroll
          for (int i = 0; i <= QMAX; ++i) s.l[i] = 0.0;
#pragma unroll
          for (int i = 0; i < 6; ++i) s.tq[i] = 0.0;
          s.saved_tq5 = 0.0;
          s.gammap = 0.0;
          s.gamrat = 1.0;
          s.gammasv = 0.0;
          s.acnrm = 0.0;
          s.crate = 1.0;
          if (bad) { s.status = ST_NONFINITE; act = A_STORE; break; }
          set_ewt(o, s, y0);
#pragma unroll
          for (int r = 0; r < R; ++r) s.yq[r] = y0[r];
          s.tq_req = o.t0;
          s.phase = PH_INIT;
          return true;
        }

        // ------------------------------------------------------ outer loop
        case A_STEP_TOP: {
          if (s.nst > 0) set_ewt(o, s, s.zn[0]);                                   // O1
          if ((s.tn + s.hprime - o.tf) * s.h > 0.0) {                              // O2
            s.hprime = o.tf - s.tn;
            s.eta = s.hprime / s.h;
          }
          if (s.nst >= o.mxstep) { s.status = ST_TOO_MUCH_WORK; act = A_STORE; break; }  // O3
          // STEP prologue
          s.saved_t = s.tn;
          s.ncf = 0;
          s.nef = 0;
          s.nflag = NF_FIRST;
          if (s.nst > 0 && s.hprime != s.h) {
            if (s.qprime != s.q) {
              adjust_order(o, s, s.qprime - s.q);
              s.q = s.qprime;
              s.L = s.q + 1;
              s.qwait = s.L;
            }
            rescale(s);
          }
          act = A_ATTEMPT;
          break;
        }
        case A_ATTEMPT: {
          predict(o, s);
          set_bdf(s);
          s.rl1 = 1.0 / s.l[1];
          s.gamma = s.h * s.rl1;
          if (s.nst == 0) s.gammap = s.gamma;
          s.gamrat = (s.nst > 0) ? s.gamma / s.gammap : 1.0;
          // NEWTON(nflag) prologue
          s.convfail = (s.nflag == NF_FIRST || s.nflag == NF_PREV_ERR) ? CF_NONE : CF_OTHER;
          s.setup = (s.nflag == NF_PREV_CONV) || (s.nflag == NF_PREV_ERR) || (s.nst == 0) ||
                    (s.nst >= s.nstlp + MSBP) || (fabs(s.gamrat - 1.0) > DGMAX);
          s.tol = s.tq[4];
          s.jcur = 0;
          act = A_REQ_RES;
          break;
        }
        case A_REQ_RES: {  // first residual of a Newton solve (ycor = 0)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            s.acor[r] = 0.0;
            s.yq[r] = s.zn[0][r];
          }
          s.m = 0;
          s.dprev = 0.0;
          s.tq_req = s.tn;
          s.phase = PH_NRES;
          return true;
        }
        case A_SOLVE: {
          s.nni++;
          double b[R];
#pragma unroll
          for (int r = 0; r < R; ++r) b[r] = -s.del[r];
          if (lsolve(g, s, LUm, perm, b)) { rv = 1; act = A_NFAIL; break; }
#pragma unroll
          for (int r = 0; r < R; ++r) s.acor[r] = s.acor[r] + b[r];
          const double del = wrms(g, b, s.ewt);
          if (s.m > 0) s.crate = fmax(CRDOWN * s.crate, del / s.dprev);
          const double dcon = del * fmin(1.0, s.crate) / s.tol;
          if (dcon <= 1.0) {
            s.acnrm = (s.m == 0) ? del : wrms(g, s.acor, s.ewt);
            act = A_ERRTEST;
            break;
          }
          if (s.m >= 1 && del > RDIV * s.dprev) { rv = 1; act = A_NFAIL; break; }
          s.dprev = del;
          s.m++;
          if (s.m >= MAXCOR) { rv = 1; act = A_NFAIL; break; }
#pragma unroll
          for (int r = 0; r < R; ++r) s.yq[r] = s.zn[0][r] + s.acor[r];
          s.tq_req = s.tn;
          s.phase = PH_NRES;
          return true;
        }
        case A_NFAIL: {
          // retry once with a fresh Jacobian/matrix if it was not current
          if (!s.jcur) {
            s.setup = 1;
            s.convfail = CF_BAD_J;
            act = A_REQ_RES;
            break;
          }
          // cvHandleNFlag: recoverable convergence failure
          s.ncfn++;
          restore(s);
          s.ncf++;
          s.etamax = 1.0;
          if (fabs(s.h) <= o.hmin * (1.0 + UROUND) || s.ncf == MXNCF) {
            s.status = ST_CONV_FAILURE;
            act = A_STORE;
            break;
          }
          s.eta = fmax(ETACF, o.hmin / fabs(s.h));
          s.nflag = NF_PREV_CONV;
          rescale(s);
          act = A_ATTEMPT;
          break;
        }
        case A_ERRTEST: {
          dsm = s.acnrm * s.tq[2];
          if (dsm <= 1.0) {
            // DONE: cvCompleteStep
            s.nst++;
#pragma unroll
            for (int i = QMAX; i >= 2; --i)
              if (i <= s.q) s.tau[i] = s.tau[i - 1];
            if (s.q == 1 && s.nst > 1) s.tau[2] = s.tau[1];
            s.tau[1] = s.h;
#pragma unroll
            for (int j = 0; j <= QMAX; ++j)
              if (j <= s.q) {
#pragma unroll
                for (int r = 0; r < R; ++r) s.zn[j][r] = s.l[j] * s.acor[r] + s.zn[j][r];
              }
            s.qwait--;
            if (s.qwait == 1 && s.q != o.qmax) {
              zn_set(s, o.qmax, s.acor);
              s.saved_tq5 = s.tq[5];
            }
            prepare_next(g, o, s, dsm);
            s.etamax = ETAMX2;
            if (fabs(s.tn - o.tf) <= 100.0 * UROUND * (fabs(s.tn) + fabs(s.h))) {   // O5
              s.tn = o.tf;
              act = A_STORE;
            } else {
              act = A_STEP_TOP;
            }
            break;
          }
          s.nef++;
          s.netf++;
          s.nflag = NF_PREV_ERR;
          restore(s);
          if (fabs(s.h) <= o.hmin * (1.0 + UROUND) || s.nef == MXNEF) {
            s.status = ST_ERR_FAILURE;
            act = A_STORE;
            break;
          }
          s.etamax = 1.0;
          if (s.nef <= MXNEF1) {
            s.eta = 1.0 / (root_l(BIAS2 * dsm, s.L) + ADDON);
            s.eta = fmax(ETAMIN, fmax(s.eta, o.hmin / fabs(s.h)));
            if (s.nef >= SMALL_NEF) s.eta = fmin(s.eta, ETAMXF);
            rescale(s);
            act = A_ATTEMPT;
            break;
          }
          if (s.q > 1) {
            s.eta = fmax(ETAMIN, o.hmin / fabs(s.h));
            adjust_order(o, s, -1);
            s.L = s.q;
            s.q = s.q - 1;
            s.qwait = s.L;
            rescale(s);
            act = A_ATTEMPT;
            break;
          }
          s.eta = fmax(ETAMIN, o.hmin / fabs(s.h));
          s.h = s.h * s.eta;
          s.hprime = s.h;
          s.hscale = s.h;
          s.qwait = LONG_WAIT;
#pragma unroll
          for (int r = 0; r < R; ++r) s.yq[r] = s.zn[0][r];
          s.tq_req = s.tn;
          s.phase = PH_ETF3;
          return true;
        }
        case A_STORE: {
          const long long c = s.cell;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int k = Lay::comp(g.lane, r);
            if (k < N && s.status != ST_NONFINITE) y[idx(o, c, k)] = s.zn[0][r];
          }
          if (g.lane == 0) {
            if (cs.status) cs.status[c] = s.status;
            if (cs.nst) cs.nst[c] = s.nst;
            if (cs.nfe) cs.nfe[c] = s.nfe;
            if (cs.nje) cs.nje[c] = s.nje;
            if (cs.nsetups) cs.nsetups[c] = s.nsetups;
            if (cs.nni) cs.nni[c] = s.nni;
            if (cs.netf) cs.netf[c] = s.netf;
            if (cs.ncfn) cs.ncfn[c] = s.ncfn;
            if (cs.q_last) cs.q_last[c] = s.q;
            if (cs.h_last) cs.h_last[c] = s.h;
            if (cs.t_reached) cs.t_reached[c] = s.tn;
            acc.n_failed += (s.status != ST_OK);
            acc.nst += s.nst;
            acc.nfe += s.nfe;
            acc.nje += s.nje;
            acc.nsetups += s.nsetups;
            acc.nni += s.nni;
            acc.netf += s.netf;
            acc.ncfn += s.ncfn;
            acc.nst_max = acc.nst_max > (unsigned long long)s.nst ? acc.nst_max : (unsigned long long)s.nst;
            acc.nfe_max = acc.nfe_max > (unsigned long long)s.nfe ? acc.nfe_max : (unsigned long long)s.nfe;
            acc.cells_done++;
          }
          act = A_LOAD;
          break;
        }
      }
    }
  }
};

template <class Model>
__global__ void __launch_bounds__(Model::BLOCK, Model::MINB) integrate_kernel(Opts o, typename Model::Params prm, double* y,
                                                                 const double* fext, const double* aux,
                                                                 const double* atol, unsigned long long* counter,
                                                                 Agg* agg, CellStatsPtrs cs) {
  using I = Integrator<Model>;
  constexpr int G = Model::G, R = I::R, N = Model::N;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5;
  double* wbase = smem + warp * I::SMEM_WARP;
  double* Jm = wbase;
  double* LUm = I::DIAG ? wbase : wbase + I::MAT;
  double* scratch = wbase + (I::DIAG ? 0 : I::MAT + I::MATLU);
  int* perm = reinterpret_cast<int*>(scratch + Model::SCRATCH);
  Grp<G> g;
  typename I::S s;
  Agg acc = {};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int k = Layout<N, G>::comp(g.lane, r);
    s.atol[r] = k < N ? atol[k] : 1.0;
  }
  s.phase = PH_DONE;
  s.cell = 0;
  s.chunk_end = 0;
  int rv = 0;
  double fr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) fr[r] = 0.0;
  bool live = true;
  for (;;) {
    if (live) live = I::advance(g, o, prm, s, rv, fr, y, fext, aux, Jm, LUm, perm, scratch, counter, acc, cs);
    if (!__any_sync(0xffffffffu, live)) break;
    if (live) {
      rv = Model::rhs(g, prm, s.tq_req, s.yq, fr, s.aux, scratch);
#pragma unroll
      for (int r = 0; r < R; ++r) fr[r] = fr[r] + s.fext[r];
      s.nfe++;
    }
  }
  // aggregate statistics: one atomic per counter per group leader
  if (g.lane == 0 && acc.cells_done) {
    atomicAdd(&agg->n_failed, acc.n_failed);
    atomicAdd(&agg->nst, acc.nst);
    atomicAdd(&agg->nfe, acc.nfe);
    atomicAdd(&agg->nje, acc.nje);
    atomicAdd(&agg->nsetups, acc.nsetups);
    atomicAdd(&agg->nni, acc.nni);
    atomicAdd(&agg->netf, acc.netf);
    atomicAdd(&agg->ncfn, acc.ncfn);
    atomicMax(&agg->nst_max, acc.nst_max);
    atomicMax(&agg->nfe_max, acc.nfe_max);
    atomicAdd(&agg->cells_done, acc.cells_done);
  }
}

}  // namespace bdfb
