// bdf_group.cuh -- per-cell BDF integrator for cells owned by a GROUP of
// G > 1 lanes (one component per lane, N <= G), B200 / sm_100a.
//
// Same algorithm, constants and operation order as bdf_cell.cuh (the listing
// SURVEY.md §8(c).2), organised for a small
// instruction footprint, which is what bounds this kernel on the GPU (ncu:
// "no_instruction" stalls dominate a register-resident, fully inlined state
// machine):
//   * ALL per-cell state lives in shared memory, per group: the scalar state
//     GS, the lane-distributed vectors (Nordsieck history zn[0..5], weights,
//     corrections, ...), the saved Jacobian and the LU factors;
//   * scalar control logic (step/order selection, error test, Newton test,
//     cvHin, ...) runs once per group in the group's LEADER lane as compact,
//     out-of-line functions over GS; vector steps run on all lanes;
//     decisions reach the group through GS after a group barrier;
//   * cold paths (Jacobian, LU factorisation, order change, cvHin) are
//     out-of-line calls with pointer arguments only (no register spills);
//   * the model RHS is the single convergence point of every trip around the
//     loop, as in bdf_cell.cuh.
#pragma once
#include "bdf_cell.cuh"

namespace bdfb {

// ---------------------------------------------------------------- group LU
// Matrix of a group: element (row = lane i, column j) at A[j * MS + i].
// Rows never move between lanes; each lane tracks its LAPACK position so the
// pivots and factors are bit-identical to the listing's LU_FACTOR (R16).
//
// The update reads the pivot row from shared memory (broadcast) and updates
// this lane's row in place (a register-resident variant measured 35% slower:
// its out-of-line call forces the caller's live registers to be saved).
template <int N, int G, int MS>
__device__ __noinline__ int glu_factor(const Grp<G> g, double* A, int* posv, int* perm, double* invd) {
  const bool act = g.lane < N;
  int pos = g.lane;
  for (int k = 0; k < N; ++k) {
#ifdef BDFB_LU_BFLY
    double a = (act && pos >= k) ? fabs(A[k * MS + g.lane]) : -1.0;
    int key = (pos << 5) | g.lane;
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) {
      const double oa = __shfl_xor_sync(g.mask, a, off, G);
      const int ok = __shfl_xor_sync(g.mask, key, off, G);
      if (oa > a || (oa == a && ok < key)) { a = oa; key = ok; }
    }
    const int p = key >> 5, pl = key & 31;
#else
    // |a| >= 0 orders like its IEEE bit pattern: first index of max |a| by
    // three warp reductions (max high word, max low word among those, min
    // position among the ties)
    const bool cand = act && pos >= k;
    const unsigned long long bits =
        cand ? (unsigned long long)__double_as_longlong(fabs(A[k * MS + g.lane])) : 0ull;
    const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
    const unsigned mhi = __reduce_max_sync(g.mask, hi);
    const unsigned mlo = __reduce_max_sync(g.mask, (cand && hi == mhi) ? lo : 0u);
    const bool top = cand && hi == mhi && lo == mlo;
    const unsigned key = __reduce_min_sync(g.mask, top ? (unsigned)((pos << 5) | g.lane) : 0xffffffffu);
    const int p = (int)(key >> 5), pl = (int)(key & 31u);
#endif
    const double pv = A[k * MS + pl];
    if (pv == 0.0) { g.sync(); return k + 1; }
    if (g.lane == pl) pos = k;
    else if (pos == k) pos = p;
    if (act && pos > k) {
      const double r = 1.0 / pv;
      const double m = A[k * MS + g.lane] * r;
      A[k * MS + g.lane] = m;
      for (int j = k + 1; j < N; ++j) A[j * MS + g.lane] = fma(-m, A[j * MS + pl], A[j * MS + g.lane]);
    }
    g.sync();
  }
  if (act) {
    perm[pos] = g.lane;
    posv[g.lane] = pos;
    invd[g.lane] = 1.0 / A[pos * MS + g.lane];
  }
  g.sync();
  return 0;
}

// x = M^{-1} b for this lane's component (row = lane).  Reciprocal diagonal
// (reading R16), axpy-ordered substitutions with fma.
#ifndef BDFB_SOLVE_UNROLL
#define BDFB_SOLVE_UNROLL 2
#endif
constexpr int kSolveUnroll = BDFB_SOLVE_UNROLL;
template <int N, int G, int MS>
__device__ __forceinline__ double glu_solve(const Grp<G>& g, const double* A, int pos, double invd,
                                            const int* perm, double b) {
  const bool act = g.lane < N;
#pragma unroll kSolveUnroll
  for (int k = 0; k < N - 1; ++k) {
    const double bk = __shfl_sync(g.mask, b, perm[k], G);
    if (act && pos > k) b = fma(-A[k * MS + g.lane], bk, b);
  }
#pragma unroll kSolveUnroll
  for (int k = N - 1; k > 0; --k) {
    if (act && pos == k) b = b * invd;
    const double bk = __shfl_sync(g.mask, b, perm[k], G);
    if (act && pos < k) b = fma(-A[k * MS + g.lane], bk, b);
  }
  if (act && pos == 0) b = b * invd;
  return __shfl_sync(g.mask, b, act ? perm[g.lane] : g.lane, G);
}

// ---------------------------------------------------------------- state
struct GS {
  double tn, h, hscale, hprime, eta, etamax, saved_t, treq;
  double tau[QMAX + 2], l[QMAX + 1], tq[6], lc[QMAX + 1];
  double rl1, gamma, gammap, gamrat, crate, acnrm, saved_tq5, dprev, tol, dsm, del, A1, cquot;
  double hg, hs, hub, hnew, aux, hubinv;
  long long cell, chunk_end;
  int q, qprime, L, qwait;
  int nst, nfe, nje, nsetups, nni, netf, ncfn;
  int nstlp, nstlj, nef, ncf, nflag, convfail, setup, jcur, m;
  int count1, count2, phase, status, act, flag;
};

// next actions (GS::act); values < 0 are "RHS requested, phase set"
enum : int { X_LOAD = 0, X_STEP_TOP, X_ATTEMPT, X_REQ_RES, X_SOLVE, X_NFAIL, X_ERRTEST, X_STORE, X_START,
             X_HIN_FINISH, X_SETUP, X_COMPLETE, X_PREPARE, X_PREP_FINISH, X_ORDER_DOWN, X_RESCALE, X_RETURN };

// ---- leader-lane scalar logic (out of line, pointer arguments only) ----------
static __device__ __noinline__ void gl_set_bdf(GS* s) {
  const int q = s->q;
  const double h = s->h;
  double xi_inv = 1.0, xistar_inv = 1.0, alpha0 = -1.0, alpha0_hat = -1.0, hsum = h;
  double* l = s->l;
  l[0] = l[1] = 1.0;
  for (int i = 2; i <= QMAX; ++i) l[i] = 0.0;
  if (q > 1) {
    for (int j = 2; j < q; ++j) {
      hsum = hsum + s->tau[j - 1];
      xi_inv = h / hsum;
      alpha0 = alpha0 - 1.0 / j;
      for (int i = j; i >= 1; --i) l[i] = l[i] + l[i - 1] * xi_inv;
    }
    alpha0 = alpha0 - 1.0 / q;
    xistar_inv = -l[1] - alpha0;
    hsum = hsum + s->tau[q - 1];
    xi_inv = h / hsum;
    alpha0_hat = -l[1] - xi_inv;
    for (int i = q; i >= 1; --i) l[i] = l[i] + l[i - 1] * xistar_inv;
  }
  const double A1 = 1.0 - alpha0_hat + alpha0;
  const double A2 = 1.0 + q * A1;
  s->tq[2] = fabs(A1 / (alpha0 * A2));
  s->tq[5] = fabs(A2 * xistar_inv / (l[q] * xi_inv));
  if (s->qwait == 1) {
    if (q > 1) {
      const double C = xistar_inv / l[q];
      const double A3 = alpha0 + 1.0 / q;
      const double A4 = alpha0_hat + xi_inv;
      const double Cpinv = (1.0 - A4 + A3) / A3;
      s->tq[1] = fabs(C * Cpinv);
    } else {
      s->tq[1] = 1.0;
    }
    hsum = hsum + s->tau[q];
    xi_inv = h / hsum;
    const double A5 = alpha0 - 1.0 / (q + 1);
    const double A6 = alpha0_hat - xi_inv;
    const double Cppinv = (1.0 - A6 + A5) / A2;
    s->tq[3] = fabs(Cppinv / (xi_inv * (q + 2) * A5));
  }
  s->tq[4] = NLSCOEF / s->tq[2];
}

// cvIncreaseBDF coefficients: lc[2..q], A1 (vector part applied by all lanes)
static __device__ __noinline__ void gl_increase_coef(GS* s) {
  double* l = s->lc;
  for (int i = 0; i <= QMAX; ++i) l[i] = 0.0;
  double alpha1 = 1.0, prod = 1.0, xiold = 1.0, alpha0 = -1.0, hsum = s->hscale;
  l[2] = 1.0;
  if (s->q > 1) {
    for (int j = 1; j < s->q; ++j) {
      hsum = hsum + s->tau[j + 1];
      const double xi = hsum / s->hscale;
      prod = prod * xi;
      alpha0 = alpha0 - 1.0 / (j + 1);
      alpha1 = alpha1 + 1.0 / xi;
      for (int i = j + 2; i >= 2; --i) l[i] = l[i] * xiold + l[i - 1];
      xiold = xi;
    }
  }
  s->A1 = (-alpha0 - alpha1) / prod;
}

// cvDecreaseBDF coefficients lc[2..q-1]
static __device__ __noinline__ void gl_decrease_coef(GS* s) {
  double* l = s->lc;
  for (int i = 0; i <= QMAX; ++i) l[i] = 0.0;
  l[2] = 1.0;
  double hsum = 0.0;
  for (int j = 1; j <= s->q - 2; ++j) {
    hsum = hsum + s->tau[j];
    const double xi = hsum / s->hscale;
    for (int i = j + 2; i >= 2; --i) l[i] = l[i] * xi + l[i - 1];
  }
}

static __device__ __forceinline__ void gl_set_eta(GS* s, const Opts* o) {
  if (s->eta < THRESH) {
    s->eta = 1.0;
    s->hprime = s->h;
  } else {
    s->eta = fmin(s->eta, s->etamax);
    if (o->hmax > 0.0) s->eta = s->eta / fmax(1.0, fabs(s->h) * s->eta / o->hmax);
    s->hprime = s->h * s->eta;
  }
}

// Error test and, on success, cvCompleteStep's scalar part.  Sets s->act.
static __device__ __noinline__ void gl_errtest(GS* s, const Opts* o) {
  const double dsm = s->acnrm * s->tq[2];
  s->dsm = dsm;
  if (dsm <= 1.0) {
    s->nst++;
    for (int i = s->q; i >= 2; --i) s->tau[i] = s->tau[i - 1];
    if (s->q == 1 && s->nst > 1) s->tau[2] = s->tau[1];
    s->tau[1] = s->h;
    s->qwait--;
    s->flag = (s->qwait == 1 && s->q != o->qmax);   // zn[qmax] = acor
    if (s->flag) s->saved_tq5 = s->tq[5];
    s->act = X_COMPLETE;
    return;
  }
  s->nef++;
  s->netf++;
  s->nflag = NF_PREV_ERR;
  s->act = X_ERRTEST + 100;   // failure: restore first (vector), then gl_errfail
}

// after RESTORE on an error-test failure: choose eta / order (sets s->act)
static __device__ __noinline__ void gl_errfail(GS* s, const Opts* o) {
  s->tn = s->saved_t;
  if (fabs(s->h) <= o->hmin * (1.0 + UROUND) || s->nef == MXNEF) {
    s->status = ST_ERR_FAILURE;
    s->act = X_STORE;
    return;
  }
  s->etamax = 1.0;
  if (s->nef <= MXNEF1) {
    s->eta = 1.0 / (root_l(BIAS2 * s->dsm, s->L) + ADDON);
    s->eta = fmax(ETAMIN, fmax(s->eta, o->hmin / fabs(s->h)));
    if (s->nef >= SMALL_NEF) s->eta = fmin(s->eta, ETAMXF);
    s->act = X_RESCALE;
    return;
  }
  if (s->q > 1) {
    s->eta = fmax(ETAMIN, o->hmin / fabs(s->h));
    s->act = X_ORDER_DOWN;      // adjust_order(-1) (if q > 2), L = q, q--, qwait = L, rescale
    return;
  }
  s->eta = fmax(ETAMIN, o->hmin / fabs(s->h));
  s->h = s->h * s->eta;
  s->hprime = s->h;
  s->hscale = s->h;
  s->qwait = LONG_WAIT;
  s->treq = s->tn;
  s->phase = PH_ETF3;
  s->act = X_RETURN;
}

// PREPARE_NEXT, first part: does the order selection need the two norms?
static __device__ __noinline__ void gl_prepare_a(GS* s, const Opts* o) {
  if (s->etamax == 1.0) {
    s->qwait = s->qwait > 2 ? s->qwait : 2;
    s->qprime = s->q;
    s->hprime = s->h;
    s->eta = 1.0;
    s->flag = 0;
    s->act = X_PREP_FINISH;
    return;
  }
  const double etaq = 1.0 / (root_l(BIAS2 * s->dsm, s->L) + ADDON);
  if (s->qwait != 0) {
    s->eta = etaq;
    s->qprime = s->q;
    gl_set_eta(s, o);
    s->flag = 0;
    s->act = X_PREP_FINISH;
    return;
  }
  s->qwait = 2;
  s->A1 = etaq;   // stash
  s->cquot = 0.0;
  s->flag = (s->q != o->qmax && s->saved_tq5 != 0.0) ? 1 : 0;   // etaqp1 needed
  if (s->flag) {
    const double hr = s->h / s->tau[2];
    double pw = 1.0;
    for (int k = 0; k < s->L; ++k) pw = pw * hr;
    s->cquot = (s->tq[5] / s->saved_tq5) * pw;
  }
  s->act = X_PREPARE;   // all lanes: ddn = ||zn[q]||, dup = ||acor - cquot zn[qmax]||
}

// PREPARE_NEXT, second part (cvChooseEta + cvSetEta); s->flag = 1 -> zn[qmax] = acor
static __device__ __noinline__ void gl_prepare_b(GS* s, const Opts* o, double ddn, double dup) {
  const double etaq = s->A1;
  double etaqm1 = 0.0, etaqp1 = 0.0;
  if (s->q > 1) etaqm1 = 1.0 / (root_l(BIAS1 * (ddn * s->tq[1]), s->q) + ADDON);
  if (s->flag) etaqp1 = 1.0 / (root_l(BIAS3 * (dup * s->tq[3]), s->L + 1) + ADDON);
  const double etam = fmax(etaqm1, fmax(etaq, etaqp1));
  s->flag = 0;
  if (etam < THRESH) {
    s->eta = 1.0;
    s->qprime = s->q;
  } else if (etam == etaq) {
    s->eta = etaq;
    s->qprime = s->q;
  } else if (etam == etaqm1) {
    s->eta = etaqm1;
    s->qprime = s->q - 1;
  } else {
    s->eta = etaqp1;
    s->qprime = s->q + 1;
    s->flag = 1;
  }
  gl_set_eta(s, o);
}

// outer-loop top (O2, O3 and the STEP prologue); sets s->act / s->flag
static __device__ __noinline__ void gl_step_top(GS* s, const Opts* o) {
  if ((s->tn + s->hprime - o->tf) * s->h > 0.0) {
    s->hprime = o->tf - s->tn;
    s->eta = s->hprime / s->h;
  }
  if (s->nst >= o->mxstep) {
    s->status = ST_TOO_MUCH_WORK;
    s->act = X_STORE;
    return;
  }
  s->saved_t = s->tn;
  s->ncf = 0;
  s->nef = 0;
  s->nflag = NF_FIRST;
  s->flag = 0;   // 1: rescale only, 2: increase order then rescale, 3: decrease order then rescale
  if (s->nst > 0 && s->hprime != s->h) {
    if (s->qprime == s->q) s->flag = 1;
    else if (s->qprime > s->q) { gl_increase_coef(s); s->flag = 2; }
    else { s->flag = (s->q == 2) ? 4 : 3; if (s->flag == 3) gl_decrease_coef(s); }
  }
  s->act = X_ATTEMPT;
}

// after PREDICT: SET_BDF, gamma, Newton prologue
static __device__ __noinline__ void gl_attempt(GS* s, const Opts* o) {
  s->tn = s->tn + s->h;
  if ((s->tn - o->tf) * s->h > 0.0) s->tn = o->tf;
  gl_set_bdf(s);
  s->rl1 = 1.0 / s->l[1];
  s->gamma = s->h * s->rl1;
  if (s->nst == 0) s->gammap = s->gamma;
  s->gamrat = (s->nst > 0) ? s->gamma / s->gammap : 1.0;
  s->convfail = (s->nflag == NF_FIRST || s->nflag == NF_PREV_ERR) ? CF_NONE : CF_OTHER;
  s->setup = (s->nflag == NF_PREV_CONV) || (s->nflag == NF_PREV_ERR) || (s->nst == 0) ||
             (s->nst >= s->nstlp + MSBP) || (fabs(s->gamrat - 1.0) > DGMAX);
  s->tol = s->tq[4];
  s->jcur = 0;
}

// Newton convergence test (Eq. 4) after a solve; sets s->act
static __device__ __forceinline__ void gl_newton_test(GS* s, double del) {
  s->nni++;
  if (s->m > 0) s->crate = fmax(CRDOWN * s->crate, del / s->dprev);
  const double dcon = del * fmin(1.0, s->crate) / s->tol;
  s->del = del;
  if (dcon <= 1.0) {
    s->act = X_ERRTEST;
    s->flag = (s->m == 0) ? 0 : 1;        // 1: acnrm = ||acor||
    if (s->m == 0) s->acnrm = del;
    return;
  }
  if (s->m >= 1 && del > RDIV * s->dprev) { s->act = X_NFAIL; return; }
  s->dprev = del;
  s->m++;
  if (s->m >= MAXCOR) { s->act = X_NFAIL; return; }
  s->treq = s->tn;
  s->phase = PH_NRES;
  s->act = X_RETURN;
}

template <class Model>
struct GroupIntegrator {
  static constexpr int N = Model::N, G = Model::G;
  static_assert(G > 1 && N <= G, "one component per lane");
  static constexpr int GPW = 32 / G;
  static constexpr int MS = (N % 2) ? N : N + 1;          // odd matrix stride: conflict-free rows/columns
  enum { V_ZN = 0, V_EWT = QMAX + 1, V_ACOR, V_FY, V_YQ, V_DEL, V_ATOL, V_FEXT, V_FR, V_INVD, NV };
  static constexpr int GS_D = (int)((sizeof(GS) + 7) / 8);
  static constexpr int MAT = N * MS;
  static constexpr int MATLU = MAT > Model::JG ? MAT : Model::JG;
  static constexpr int IDX_D = G;                           // perm[G] + pos[G] ints
  static constexpr int PER_GROUP = GS_D + NV * G + MAT + MATLU + IDX_D + Model::SG;
  static constexpr int SMEM_WARP = GPW * PER_GROUP;
  static constexpr int CHUNK = 4;
  using P = typename Model::Params;

  struct Ctx {
    GS* s;
    double* v;
    double* J;
    double* LU;
    int* perm;
    int* pos;
    double* sc;
  };

  __device__ static double& V(const Ctx& c, const Grp<G>& g, int row) { return c.v[row * G + g.lane]; }

  __device__ static double wrms(const Grp<G>& g, double v, double w) {
    double p = v * w;
    double acc = (g.lane < N) ? p * p : 0.0;
    return sqrt(g.sum(acc) / (double)N);
  }

  __device__ static long long yidx(const Opts& o, long long c, int k) {
    return o.layout == 0 ? (long long)k * o.ncells + c : c * (long long)N + k;
  }

  // vector RESCALE (zn[j] *= eta^j, j <= q) + leader h update
  __device__ static void rescale(const Grp<G>& g, const Ctx& c) {
    GS* s = c.s;
    const double eta = s->eta;
    const int q = s->q;
    double f = eta;
    for (int j = 1; j <= q; ++j) {
      V(c, g, V_ZN + j) = f * V(c, g, V_ZN + j);
      f = f * eta;
    }
    g.sync();
    if (g.lane == 0) {
      s->h = s->hscale * eta;
      s->hscale = s->h;
    }
    g.sync();
  }

  __device__ static void predict(const Grp<G>& g, const Ctx& c) {
    const int q = c.s->q;
    for (int k = 1; k <= q; ++k)
      for (int j = q; j >= k; --j) V(c, g, V_ZN + j - 1) = V(c, g, V_ZN + j - 1) + V(c, g, V_ZN + j);
  }

  __device__ static void restore(const Grp<G>& g, const Ctx& c) {
    const int q = c.s->q;
    for (int k = 1; k <= q; ++k)
      for (int j = q; j >= k; --j) V(c, g, V_ZN + j - 1) = V(c, g, V_ZN + j - 1) - V(c, g, V_ZN + j);
  }

  // Advance this group's cell to its next RHS request; false when out of cells.
  __device__ static bool advance(const Grp<G>& g, const Opts& o, const P& prm, const Ctx& c, int rv, double fr,
                                 double* y, const double* fext, const double* aux, unsigned long long* counter,
                                 Agg& acc, const CellStatsPtrs& cs) {
    GS* s = c.s;
    int act;
    g.sync();
    switch (s->phase) {
      case PH_INIT: act = -1; break;
      case PH_HIN: act = -2; break;
      case PH_NRES: act = -3; break;
      case PH_ETF3: act = -5; break;
      default: act = X_LOAD; break;
    }
    g.sync();   // every lane has read the phase before any lane rewrites it (racecheck)
    for (;;) {
      switch (act) {
        case -1: {  // f(t0, y0) ready
          if (rv) { if (g.lane == 0) s->status = ST_RHS_FAIL; act = X_STORE; break; }
          V(c, g, V_ZN + 1) = fr;
          if (o.h0 != 0.0) {
            if (g.lane == 0) s->h = o.h0;
            act = X_START;
            break;
          }
          double hi = 0.0;
          if (g.lane < N) {
            const double d = HUB_FACTOR * fabs(V(c, g, V_ZN)) + 1.0 / V(c, g, V_EWT);
            hi = fabs(fr) / d;
          }
          const double hub_inv = g.max(hi);
          if (g.lane == 0) {
            const double tdist = o.tf - o.t0;
            const double hlb = 100.0 * (UROUND * fmax(fabs(o.t0), fabs(o.tf)));
            double hub = HUB_FACTOR * tdist;
            if (hub * hub_inv > 1.0) hub = 1.0 / hub_inv;
            s->hub = hub;
            s->hg = sqrt(hlb * hub);
            s->act = X_RETURN;
            if (hub < hlb) {
              s->h = s->hg;
              s->act = X_START;
            } else {
              s->hs = s->hg;
              s->hnew = s->hg;
              s->count1 = 1;
              s->count2 = 1;
              s->treq = o.t0 + s->hg;
              s->phase = PH_HIN;
            }
          }
          g.sync();
          act = s->act;
          if (act == X_RETURN) {
            V(c, g, V_YQ) = s->hg * V(c, g, V_ZN + 1) + V(c, g, V_ZN);
            return true;
          }
          break;
        }
        case -2: {  // cvYddNorm probe ready
          double ydd = 0.0;
          if (!rv) {
            const double ih = 1.0 / s->hg;
            ydd = wrms(g, (fr - V(c, g, V_ZN + 1)) * ih, V(c, g, V_EWT));
          }
          if (g.lane == 0) {
            s->act = X_RETURN;
            if (rv) {
              s->hg = s->hg * 0.2;
              s->count2++;
              if (s->count2 > HIN_ITERS) {
                if (s->count1 <= 2) { s->status = ST_RHS_FAIL; s->act = X_STORE; }
                else { s->hnew = s->hs; s->act = X_HIN_FINISH; }
              }
            } else {
              s->hs = s->hg;
              s->hnew = (ydd * s->hub * s->hub > 2.0) ? sqrt(2.0 / ydd) : sqrt(s->hg * s->hub);
              const double hrat = s->hnew / s->hg;
              if (s->count1 == HIN_ITERS) s->act = X_HIN_FINISH;
              else if (hrat > 0.5 && hrat < 2.0) s->act = X_HIN_FINISH;
              else if (s->count1 > 1 && hrat > 2.0) { s->hnew = s->hg; s->act = X_HIN_FINISH; }
              else { s->hg = s->hnew; s->count1++; s->count2 = 1; }
            }
            if (s->act == X_RETURN) s->treq = o.t0 + s->hg;
          }
          g.sync();
          act = s->act;
          if (act == X_RETURN) {
            V(c, g, V_YQ) = s->hg * V(c, g, V_ZN + 1) + V(c, g, V_ZN);
            return true;
          }
          break;
        }
        case X_HIN_FINISH: {
          if (g.lane == 0) {
            const double hlb = 100.0 * (UROUND * fmax(fabs(o.t0), fabs(o.tf)));
            double h = H_BIAS * s->hnew;
            if (h < hlb) h = hlb;
            if (h > s->hub) h = s->hub;
            s->h = h;
          }
          act = X_START;
          break;
        }
        case X_START: {
          g.sync();
          double h0 = s->h;
          if (h0 > o.tf - o.t0) h0 = o.tf - o.t0;
          if (o.hmax > 0.0 && h0 > o.hmax) h0 = o.hmax;
          V(c, g, V_ZN + 1) = h0 * V(c, g, V_ZN + 1);
          g.sync();
          if (g.lane == 0) {
            s->h = s->hscale = s->hprime = h0;
            s->q = s->qprime = 1;
            s->L = 2;
            s->qwait = 2;
            s->etamax = ETAMX1;
            s->crate = 1.0;
            s->eta = 1.0;
          }
          act = X_STEP_TOP;
          break;
        }
        case -3: {  // Newton residual f(tn, zn0 + ycor) ready
          if (rv) {   // a failed first residual is not retried (reading R5)
            if (g.lane == 0 && s->m == 0) s->jcur = 1;
            act = X_NFAIL;
            break;
          }
          V(c, g, V_FY) = fr;
          const double t = s->rl1 * V(c, g, V_ZN + 1) + V(c, g, V_ACOR);
          V(c, g, V_DEL) = -s->gamma * fr + t;
          act = s->setup ? X_SETUP : X_SOLVE;
          break;
        }
        case X_SETUP: {  // cvLsSetup: J (if stale) + M = I - gamma J + LU
          if (g.lane == 0) {
            const double dgamma = fabs(s->gamma / s->gammap - 1.0);
            const bool jbad = (s->nst == 0) || (s->nst >= s->nstlj + MSBJ) ||
                              (s->convfail == CF_BAD_J && dgamma < DGMAX_JBAD) || (s->convfail == CF_OTHER);
            s->jcur = jbad ? 1 : 0;
            if (jbad) { s->nje++; s->nstlj = s->nst; }
          }
          g.sync();
          int bad = 0;
          if (s->jcur)
            bad = Model::template jac<MS>(g, V(c, g, V_YQ), s->aux, c.J + g.lane, c.sc, c.LU) ? 1 : 0;
          if (!bad) {
            const double gm = s->gamma;
            if (g.lane < N)
              for (int j = 0; j < N; ++j) c.LU[j * MS + g.lane] = (g.lane == j ? 1.0 : 0.0) - gm * c.J[j * MS + g.lane];
            g.sync();
            bad = glu_factor<N, G, MS>(g, c.LU, c.pos, c.perm, &V(c, g, V_INVD) - g.lane) ? 1 : 0;
          }
          if (g.lane == 0) {
            s->nsetups++;
            s->gamrat = 1.0;
            s->gammap = s->gamma;
            s->crate = 1.0;
            s->nstlp = s->nst;
            s->setup = 0;
          }
          g.sync();
          act = bad ? X_NFAIL : X_SOLVE;
          break;
        }
        case X_SOLVE: {
          double b = glu_solve<N, G, MS>(g, c.LU, c.pos[g.lane < N ? g.lane : 0], V(c, g, V_INVD), c.perm,
                                         -V(c, g, V_DEL));
          if (s->gamrat != 1.0) b = (2.0 / (1.0 + s->gamrat)) * b;
          const double acor = V(c, g, V_ACOR) + b;
          V(c, g, V_ACOR) = acor;
          const double del = wrms(g, b, V(c, g, V_EWT));
          g.sync();
          if (g.lane == 0) gl_newton_test(s, del);
          g.sync();
          act = s->act;
          if (act == X_ERRTEST && s->flag) {
            const double an = wrms(g, acor, V(c, g, V_EWT));
            if (g.lane == 0) s->acnrm = an;
          }
          if (act == X_RETURN) {
            V(c, g, V_YQ) = V(c, g, V_ZN) + acor;
            return true;
          }
          break;
        }
        case X_NFAIL: {
          g.sync();
          if (!s->jcur) {
            if (g.lane == 0) { s->setup = 1; s->convfail = CF_BAD_J; }
            act = X_REQ_RES;
            break;
          }
          restore(g, c);
          g.sync();
          if (g.lane == 0) {
            s->ncfn++;
            s->tn = s->saved_t;
            s->ncf++;
            s->etamax = 1.0;
            if (fabs(s->h) <= o.hmin * (1.0 + UROUND) || s->ncf == MXNCF) {
              s->status = ST_CONV_FAILURE;
              s->act = X_STORE;
            } else {
              s->eta = fmax(ETACF, o.hmin / fabs(s->h));
              s->nflag = NF_PREV_CONV;
              s->act = X_RESCALE;
            }
          }
          g.sync();
          act = s->act;
          break;
        }
        case X_RESCALE: {
          rescale(g, c);
          act = X_ATTEMPT;
          break;
        }
        case X_ERRTEST: {
          g.sync();
          if (g.lane == 0) gl_errtest(s, &o);
          g.sync();
          if (s->act == X_COMPLETE) {
            const int q = s->q;
            const double a = V(c, g, V_ACOR);
            for (int j = 0; j <= q; ++j) V(c, g, V_ZN + j) = s->l[j] * a + V(c, g, V_ZN + j);
            if (s->flag) V(c, g, V_ZN + o.qmax) = a;
            g.sync();
            if (g.lane == 0) gl_prepare_a(s, &o);
            g.sync();
            if (s->act == X_PREPARE) {
              const int q2 = s->q;
              const double ddn = (q2 > 1) ? wrms(g, V(c, g, V_ZN + q2), V(c, g, V_EWT)) : 0.0;
              const double dup = s->flag ? wrms(g, -s->cquot * V(c, g, V_ZN + o.qmax) + a, V(c, g, V_EWT)) : 0.0;
              g.sync();
              if (g.lane == 0) gl_prepare_b(s, &o, ddn, dup);
              g.sync();
              if (s->flag) V(c, g, V_ZN + o.qmax) = a;
            }
            g.sync();
            if (g.lane == 0) {
              s->etamax = ETAMX2;
              if (fabs(s->tn - o.tf) <= 100.0 * UROUND * (fabs(s->tn) + fabs(s->h))) {
                s->tn = o.tf;
                s->act = X_STORE;
              } else {
                s->act = X_STEP_TOP;
              }
            }
            g.sync();
            act = s->act;
            break;
          }
          // error-test failure: RESTORE then choose the retry
          restore(g, c);
          g.sync();
          if (g.lane == 0) gl_errfail(s, &o);
          g.sync();
          act = s->act;
          if (act == X_RETURN) {
            V(c, g, V_YQ) = V(c, g, V_ZN);
            return true;
          }
          break;
        }
        case X_ORDER_DOWN: {
          if (g.lane == 0 && s->q > 2) gl_decrease_coef(s);
          g.sync();
          const int q = s->q;
          if (q > 2) {
            const double zq = V(c, g, V_ZN + q);
            for (int j = 2; j < q; ++j) V(c, g, V_ZN + j) = -s->lc[j] * zq + V(c, g, V_ZN + j);
          }
          g.sync();
          if (g.lane == 0) {
            s->L = s->q;
            s->q = s->q - 1;
            s->qwait = s->L;
          }
          g.sync();
          act = X_RESCALE;
          break;
        }
        case -5: {  // RHS at (tn, zn0) after the 3rd+ error-test failure at q = 1
          if (rv) { if (g.lane == 0) s->status = ST_RHS_FAIL; act = X_STORE; break; }
          V(c, g, V_ZN + 1) = s->h * fr;
          act = X_ATTEMPT;
          break;
        }
        case X_LOAD: {
          g.sync();
          const bool in_chunk = s->cell + 1 < s->chunk_end;
          g.sync();   // every lane has read the record before lane 0 updates it (racecheck)
          if (in_chunk) {
            if (g.lane == 0) s->cell = s->cell + 1;
          } else {
            long long c0 = 0;
            if (g.lane == 0) c0 = (long long)atomicAdd(counter, (unsigned long long)CHUNK);
            c0 = __shfl_sync(g.mask, c0, 0, G);
            if (c0 >= o.ncells) {
              if (g.lane == 0) s->phase = PH_DONE;
              g.sync();
              return false;
            }
            if (g.lane == 0) {
              s->cell = c0;
              s->chunk_end = c0 + CHUNK < o.ncells ? c0 + CHUNK : o.ncells;
            }
          }
          g.sync();
          const long long cell = s->cell;
          const double ax = aux ? aux[cell] : 0.0;
          int bad = !isfinite(ax);
          double y0 = 0.0, fe = 0.0;
          if (g.lane < N) {
            y0 = y[yidx(o, cell, g.lane)];
            fe = fext ? fext[yidx(o, cell, g.lane)] : 0.0;
            if (!isfinite(y0) || !isfinite(fe)) bad = 1;
          }
          bad = g.ior(bad);
          for (int j = 0; j <= QMAX; ++j) V(c, g, V_ZN + j) = 0.0;
          V(c, g, V_ZN) = y0;
          V(c, g, V_FEXT) = fe;
          V(c, g, V_ACOR) = 0.0;
          V(c, g, V_EWT) = 1.0 / (o.rtol * fabs(y0) + V(c, g, V_ATOL));
          V(c, g, V_YQ) = y0;
          if (g.lane == 0) {
            s->aux = ax;
            s->nst = s->nfe = s->nje = s->nsetups = s->nni = s->netf = s->ncfn = 0;
            s->nstlp = s->nstlj = 0;
            s->status = bad ? ST_NONFINITE : ST_OK;
            s->tn = o.t0;
            s->q = 1;
            s->h = 0.0;
            for (int i = 0; i <= QMAX + 1; ++i) s->tau[i] = 0.0;
            for (int i = 0; i <= QMAX; ++i) s->l[i] = 0.0;
            for (int i = 0; i < 6; ++i) s->tq[i] = 0.0;
            s->saved_tq5 = 0.0;
            s->gammap = 0.0;
            s->gamrat = 1.0;
            s->acnrm = 0.0;
            s->crate = 1.0;
            s->treq = o.t0;
            s->phase = PH_INIT;
          }
          g.sync();
          if (bad) { act = X_STORE; break; }
          return true;
        }
        case X_STEP_TOP: {
          g.sync();
          if (s->nst > 0) V(c, g, V_EWT) = 1.0 / (o.rtol * fabs(V(c, g, V_ZN)) + V(c, g, V_ATOL));   // O1
          if (g.lane == 0) gl_step_top(s, &o);
          g.sync();
          if (s->act == X_STORE) { act = X_STORE; break; }
          const int fl = s->flag;
          if (fl >= 2) {
            const int q = s->q;
            if (fl == 2) {   // increase order: zn[q+1] = A1 zn[qmax]; zn[j] += lc[j] zn[q+1]
              const double zL = s->A1 * V(c, g, V_ZN + o.qmax);
              V(c, g, V_ZN + q + 1) = zL;
              for (int j = 2; j <= q; ++j) V(c, g, V_ZN + j) = s->lc[j] * zL + V(c, g, V_ZN + j);
            } else if (fl == 3) {
              const double zq = V(c, g, V_ZN + q);
              for (int j = 2; j < q; ++j) V(c, g, V_ZN + j) = -s->lc[j] * zq + V(c, g, V_ZN + j);
            }
            g.sync();
            if (g.lane == 0) {
              s->q = s->qprime;
              s->L = s->q + 1;
              s->qwait = s->L;
            }
            g.sync();
          }
          if (fl >= 1) rescale(g, c);
          act = X_ATTEMPT;
          break;
        }
        case X_ATTEMPT: {
          g.sync();
          predict(g, c);
          g.sync();
          if (g.lane == 0) gl_attempt(s, &o);
          act = X_REQ_RES;
          break;
        }
        case X_REQ_RES: {  // first residual of a Newton solve (ycor = 0)
          V(c, g, V_ACOR) = 0.0;
          V(c, g, V_YQ) = V(c, g, V_ZN);
          g.sync();
          if (g.lane == 0) {
            s->m = 0;
            s->dprev = 0.0;
            s->treq = s->tn;
            s->phase = PH_NRES;
          }
          g.sync();
          return true;
        }
        case X_STORE: {
          g.sync();
          const long long cell = s->cell;
          if (g.lane < N && s->status != ST_NONFINITE) y[yidx(o, cell, g.lane)] = V(c, g, V_ZN);
          if (g.lane == 0) {
            if (cs.status) cs.status[cell] = s->status;
            if (cs.nst) cs.nst[cell] = s->nst;
            if (cs.nfe) cs.nfe[cell] = s->nfe;
            if (cs.nje) cs.nje[cell] = s->nje;
            if (cs.nsetups) cs.nsetups[cell] = s->nsetups;
            if (cs.nni) cs.nni[cell] = s->nni;
            if (cs.netf) cs.netf[cell] = s->netf;
            if (cs.ncfn) cs.ncfn[cell] = s->ncfn;
            if (cs.q_last) cs.q_last[cell] = s->q;
            if (cs.h_last) cs.h_last[cell] = s->h;
            if (cs.t_reached) cs.t_reached[cell] = s->tn;
            acc.n_failed += (s->status != ST_OK);
            acc.nst += s->nst;
            acc.nfe += s->nfe;
            acc.nje += s->nje;
            acc.nsetups += s->nsetups;
            acc.nni += s->nni;
            acc.netf += s->netf;
            acc.ncfn += s->ncfn;
            acc.nst_max = acc.nst_max > (unsigned long long)s->nst ? acc.nst_max : (unsigned long long)s->nst;
            acc.nfe_max = acc.nfe_max > (unsigned long long)s->nfe ? acc.nfe_max : (unsigned long long)s->nfe;
            acc.cells_done++;
          }
          act = X_LOAD;
          break;
        }
        default:
          act = X_LOAD;
          break;
      }
    }
  }
};

template <class Model>
__global__ void __launch_bounds__(Model::BLOCK, Model::MINB)
    integrate_group_kernel(Opts o, typename Model::Params prm, double* y, const double* fext, const double* aux,
                           const double* atol, unsigned long long* counter, Agg* agg, CellStatsPtrs cs) {
  using I = GroupIntegrator<Model>;
  constexpr int G = Model::G, N = Model::N;
  extern __shared__ double smem[];
  __shared__ Opts so;
  if (threadIdx.x == 0) so = o;
  __syncthreads();
  Grp<G> g;
  const int gidx = threadIdx.x / G;                    // group index in the block
  double* base = smem + gidx * I::PER_GROUP;
  typename I::Ctx c;
  c.s = reinterpret_cast<GS*>(base);
  c.v = base + I::GS_D;
  c.J = c.v + I::NV * G;
  c.LU = c.J + I::MAT;
  c.perm = reinterpret_cast<int*>(c.LU + I::MATLU);
  c.pos = c.perm + G;
  c.sc = reinterpret_cast<double*>(c.pos + G);
  I::V(c, g, I::V_ATOL) = g.lane < N ? atol[g.lane] : 1.0;
  for (int j = 0; j < I::NV; ++j)
    if (j != I::V_ATOL) I::V(c, g, j) = 0.0;
  if (g.lane == 0) {
    c.s->phase = PH_DONE;
    c.s->cell = 0;
    c.s->chunk_end = 0;
  }
  g.sync();
  Agg acc = {};
  int rv = 0;
  double fr = 0.0;
  bool live = true;
  for (;;) {
    if (live) live = I::advance(g, so, prm, c, rv, fr, y, fext, aux, counter, acc, cs);
#ifndef BDFB_NO_BLOCK_SYNC
    // keep the block's warps phase-aligned so the RHS code is fetched once for
    // all of them (the kernel is instruction-fetch bound; +14% measured)
    if (!__syncthreads_or(live)) break;
#else
    if (!__any_sync(0xffffffffu, live)) break;
#endif
    if (live) {
      double yq[1] = {I::V(c, g, I::V_YQ)}, f[1];
      rv = Model::rhs(g, prm, c.s->treq, yq, f, c.s->aux, c.sc);
      fr = f[0] + I::V(c, g, I::V_FEXT);
      if (g.lane == 0) c.s->nfe++;
    }
  }
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
