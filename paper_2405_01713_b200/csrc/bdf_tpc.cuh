// bdf_tpc.cuh -- thread-per-cell BDF integrator for the reacting-flow
// mechanism models (H2/air n = 10, DRM19-class n = 22), B200 / sm_100a.
//
// Semantics: the listing SURVEY.md §8(c).2 (CVODE's fixed-leading-coefficient
// Nordsieck BDF, orders 1..5), with the
// same state machine, constants and operation order as bdf_cell.cuh (no code
// shared with oracle/).  Organisation for the GPU:
//
//  * ONE CELL PER THREAD.  A warp advances 32 independent cells; lanes whose
//    cells are in different phases (setup / no setup, different order, a
//    retry) are masked, which is the north_star's "per-cell adaptive stepping
//    with masked lanes".  Every lane does its own cell's whole RHS (the
//    generated straight-line code of gen/tpc_<mech>.cuh: no table loads, no
//    shuffles, no group barriers), so the FP64 pipe sees full warps.
//  * The scalar state of a cell (h, q, tau, l, tq, counters, ...) lives in
//    SHARED memory, one odd-stride record per thread (bank-conflict free).
//  * The cell's vectors (Nordsieck zn[0..5], weights, corrections), the saved
//    Jacobian, the LU factors and the pivot order live in a per-thread-slot
//    WORKSPACE in device memory, element-major across slots
//    (w[e * S + slot]): every warp access is one coalesced 256-byte line pair,
//    served by L1/L2.  The workspace is sized for the resident grid only
//    (persistent kernel), not for the cell count.
//  * Matrix setup fuses M = I - gamma J into a left-looking LU with partial
//    pivoting: the column being factored stays in registers, the L entries
//    are read once per later column, the pivot search is a register compare
//    chain.  Every element receives the listing's right-looking fma sequence
//    (k increasing), so pivots and factors are bit-identical to LU_FACTOR.
//  * The solve gathers the right-hand side in pivot order and runs the unit-L
//    forward and reciprocal-diagonal back substitution in registers (R16).
//  * The model RHS is the single convergence point of every trip around the
//    loop, as in bdf_cell.cuh; blocks stay trip-aligned (__syncthreads_or) so
//    the warps of a block stream the same straight-line code together.
//
// WRMS summation order (reading R15) for G = 1: sequential in increasing i.
#pragma once
#include "bdf_cell.cuh"

namespace bdfb {

// scalar state of one cell (shared memory)
struct TS {
  double tn, tq_req, h, hscale, hprime, eta, etamax, saved_t;
  double tau[QMAX + 2], l[QMAX + 1], tq[6];
  double rl1, gamma, gammap, gamrat, crate, acnrm, saved_tq5, dprev, tol;
  double hg, hs, hub, hnew, aux, rs_eta;
  double oc_a1;                                    // deferred order increase: cvIncreaseBDF's A1
  long long cell;
  int nst, nfe, nje, nsetups, nni, netf, ncfn, nstlp, nstlj;
  // small counters and codes as bytes: the record is staged through shared memory by the SPLIT control
  // kernel, whose occupancy its size bounds (51 doubles: 4 blocks of 128 threads per SM)
  signed char q, qprime, L, qwait, nef, ncf, nflag, convfail, setup, jcur, m, count1, count2, phase, status;
  signed char flag;                                // ATTEMPT-pass flags (F_*)
  signed char coop;                                // result of a cooperative/separate stage (J, LU status)
  signed char pend;                                // split kernel: setup stage requested (A_SETUP_J/LU)
  signed char qc;                                  // order of the step whose completion is deferred (F_COMPLETE)
};
constexpr int TS_STRIDE = (int)((sizeof(TS) + 7) / 8) | 1;   // odd number of doubles
// chunks (CH elements of every Nordsieck row) of the ATTEMPT pass in flight: measured on C4 K_ctl (same box, two
// runs each): 1 -> 3151 ms, 2 -> 3295 ms, 4 -> 3709 ms (more rows in flight per lane only add L1/L2 queueing to a
// kernel whose lanes already stream ~10 KB per trip; profiles/r2/history.md)
#ifndef BDFB_ATTEMPT_UNROLL
#define BDFB_ATTEMPT_UNROLL 1
#endif
constexpr int kAttemptUnroll = BDFB_ATTEMPT_UNROLL;
// elements per ATTEMPT chunk (0: 4 when 4 divides n, else 2); 1 measured on C4 K_ctl: 3155 -> 3106 ms
#ifndef BDFB_ATTEMPT_CH
#define BDFB_ATTEMPT_CH 1
#endif
// components of the error test's PREPARE_NEXT norms per round of loads (11: 2 rounds for n = 22)
#ifndef BDFB_ERRTEST_UNROLL
#define BDFB_ERRTEST_UNROLL 11
#endif
constexpr int kErrtestUnroll = BDFB_ERRTEST_UNROLL;

#ifndef BDFB_TPC_BLOCK
#define BDFB_TPC_BLOCK 128
#endif
#ifndef BDFB_TPC_MINB
#define BDFB_TPC_MINB 2
#endif
// LU stage organisation: 0 block-packed thread-per-cell (default), 1 warp-cooperative
// per cell, 2 thread-per-cell in place (experiments; identical results)
// set_bdf (every attempt) and prepare_next (every step): out of line by default (register budget of the
// control kernels); BDFB_HOT_INLINE_ON=1 inlines them (the call saves/restores live registers through local
// memory: 517 STL/LDL in K_ctl's SASS)
#if defined(BDFB_HOT_INLINE_ON) && BDFB_HOT_INLINE_ON
#define BDFB_HOT_INLINE __forceinline__
#else
#define BDFB_HOT_INLINE __noinline__
#endif

#ifndef BDFB_TPC_LU
#define BDFB_TPC_LU 0
#endif

// per-thread-slot workspace, blocked by CTA: element e of thread t of block b at
// ws[(b * DOUBLES + e) * BLOCK + t].  A warp access to one element is one
// coalesced 256-byte line pair, and every element offset is a compile-time
// immediate (e * BLOCK * 8 bytes) from ONE base pointer per thread -- no
// per-element address registers (which otherwise spill).
template <int N, long long SS = BDFB_TPC_BLOCK, bool MATS = true>
struct TWs {
  static constexpr int O_ZN = 0, O_EWT = (QMAX + 1) * N, O_ACOR = O_EWT + N, O_YQ = O_ACOR + N, O_DEL = O_YQ + N,
                       O_FEXT = O_DEL + N, O_INVD = O_FEXT + N, O_FR = O_INVD + N, O_J = O_FR + N,
                       O_LU = O_J + N * N, DOUBLES = MATS ? O_LU + N * N : O_J, INTS = MATS ? N : 0;
  static constexpr long long S = SS;
  double* w;
  int* iw;
  __device__ __forceinline__ double& at(int e) const { return w[(long long)e * S]; }
  __device__ __forceinline__ double& zn(int j, int i) const { return at(O_ZN + j * N + i); }
  __device__ __forceinline__ double& ewt(int i) const { return at(O_EWT + i); }
  __device__ __forceinline__ double& acor(int i) const { return at(O_ACOR + i); }
  __device__ __forceinline__ double& yq(int i) const { return at(O_YQ + i); }
  __device__ __forceinline__ double& del(int i) const { return at(O_DEL + i); }
  __device__ __forceinline__ double& fext(int i) const { return at(O_FEXT + i); }
  __device__ __forceinline__ double& invd(int i) const { return at(O_INVD + i); }
  __device__ __forceinline__ double& fr(int i) const { return at(O_FR + i); }
  __device__ __forceinline__ double& J(int i, int j) const { return at(O_J + i * N + j); }
  __device__ __forceinline__ double& LU(int i, int j) const { return at(O_LU + i * N + j); }
  __device__ __forceinline__ int& perm(int i) const { return iw[(long long)i * S]; }
};

// ---------------------------------------------------------------- linear algebra
// M = I - gamma J fused into a left-looking LU with partial pivoting (listing
// LU_FACTOR, reading R16).  Returns 0, or k+1 for an exact zero pivot in
// column k (recoverable).  On success LU holds the factors in pivoted row
// positions, perm[i] = original row at position i, invd[i] = 1/U[i][i].
// piv (optional, diagnostics): LAPACK-style pivot indices.
// FORM_M = false factors the given matrix itself (diagnostic entry point; Jp may
// alias LUp: column j is read before any column >= j is written).
// SS: compile-time element stride (0 = the runtime stride Srt).  CM: J and LU
// column-major ((i, j) at element j * N + i) instead of row-major.
template <int N, bool FORM_M, long long SS, bool CM = false>
__device__ __noinline__ int tpc_factor(const double* Jp, double* LUp, double* __restrict__ invdp,
                                       int* __restrict__ permp, long long Srt, double gamma, int* __restrict__ pivp) {
  const long long S = SS ? SS : Srt;
  auto J = [&](int i, int j) -> const double& { return Jp[(long long)(CM ? j * N + i : i * N + j) * S]; };
  auto LU = [&](int i, int j) -> double& { return LUp[(long long)(CM ? j * N + i : i * N + j) * S]; };
  int perm[N];
#pragma unroll
  for (int i = 0; i < N; ++i) perm[i] = i;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double col[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int r = perm[i];
      col[i] = FORM_M ? (r == j ? 1.0 : 0.0) - gamma * J(r, j) : J(r, j);
    }
    // updates from the already factored columns k < j (same fma order as the
    // right-looking listing: k increasing for every element)
#pragma unroll
    for (int k = 0; k < j; ++k) {
      const double ukj = col[k];
#pragma unroll
      for (int i = k + 1; i < N; ++i) col[i] = fma(-LU(i, k), ukj, col[i]);
    }
    // first index of max |col[i]|, i >= j
    int p = j;
    double amax = fabs(col[j]);
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      const double a = fabs(col[i]);
      if (a > amax) { amax = a; p = i; }
    }
    if (pivp) pivp[(long long)j * S] = p;
    if (amax == 0.0) return j + 1;   // |pivot| = amax (listing: M[p][k] == 0 is singular)
    if (p != j) {
      // interchange rows j and p: branch-free selects keep col[] and perm[] in registers
      const double cj = col[j];
      const int rj = perm[j];
      double nj = cj;
      int nr = rj;
#pragma unroll
      for (int i = j + 1; i < N; ++i) {
        const bool hit = (i == p);
        nj = hit ? col[i] : nj;
        nr = hit ? perm[i] : nr;
        col[i] = hit ? cj : col[i];
        perm[i] = hit ? rj : perm[i];
      }
      col[j] = nj;
      perm[j] = nr;
      for (int k = 0; k < j; ++k) {   // swap the L parts of rows j and p
        const double t = LU(j, k);
        LU(j, k) = LU(p, k);
        LU(p, k) = t;
      }
    }
#pragma unroll
    for (int i = 0; i <= j; ++i) LU(i, j) = col[i];
    const double r = 1.0 / col[j];
    invdp[(long long)j * S] = r;
#pragma unroll
    for (int i = j + 1; i < N; ++i) LU(i, j) = col[i] * r;
    asm volatile("" ::: "memory");   // one column in flight: bounds register pressure
  }
#pragma unroll
  for (int i = 0; i < N; ++i) permp[(long long)i * S] = perm[i];
  return 0;
}

// x = M^{-1} b with b = -del (listing LU_SOLVE: row interchanges, unit-L
// forward substitution in column (axpy) order, back substitution multiplying
// by the correctly rounded 1/U[k][k], reading R16).
// b (stride S, natural order; negated first if NEG) -> x in registers.
template <int N, bool NEG, long long SS>
__device__ __forceinline__ void tpc_solve(const double* __restrict__ LUp, const double* __restrict__ invdp,
                                          const int* __restrict__ permp, const double* __restrict__ bp, long long Srt,
                                          double (&x)[N]) {
  const long long S = SS ? SS : Srt;
  auto LU = [&](int i, int j) -> const double& { return LUp[(long long)(i * N + j) * S]; };
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double v = bp[(long long)permp[(long long)i * S] * S];
    x[i] = NEG ? -v : v;
  }
#pragma unroll
  for (int k = 0; k < N - 1; ++k) {
#pragma unroll
    for (int i = k + 1; i < N; ++i) x[i] = fma(-LU(i, k), x[k], x[i]);
    if (k % 4 == 3) asm volatile("" ::: "memory");   // bounded load hoisting (register pressure)
  }
#pragma unroll
  for (int k = N - 1; k > 0; --k) {
    x[k] = x[k] * invdp[(long long)k * S];
#pragma unroll
    for (int i = 0; i < k; ++i) x[i] = fma(-LU(i, k), x[k], x[i]);
    if (k % 4 == 0) asm volatile("" ::: "memory");
  }
  x[0] = x[0] * invdp[0];
}


// Warp-cooperative LU with partial pivoting of ONE cell by a group of G lanes,
// lane i < N holding row i in registers: the listing's LU_FACTOR (reading R16:
// first index of max |.| via three redux reductions on the IEEE bits, exact
// zero pivot = singular, reciprocal-multiply column scaling, fma updates), so
// pivots and factors are bit-identical to tpc_factor / the oracle.  pos: the
// row's position in the pivoted factor; dinv: 1/U[pos][pos], set by the lane
// when its row becomes the pivot row.  Returns 0, or k+1 (group-uniform).
template <int N, int G>
__device__ __forceinline__ int coop_factor(const Grp<G>& g, double (&row)[N], int& pos, double& dinv) {
  const bool act = g.lane < N;
  pos = g.lane;
  dinv = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const bool cand = act && pos >= k;
    const unsigned long long bits = cand ? (unsigned long long)__double_as_longlong(fabs(row[k])) : 0ull;
    const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
    const unsigned mhi = __reduce_max_sync(g.mask, hi);
    const unsigned mlo = __reduce_max_sync(g.mask, (cand && hi == mhi) ? lo : 0u);
    const bool top = cand && hi == mhi && lo == mlo;
    const unsigned key = __reduce_min_sync(g.mask, top ? (unsigned)((pos << 5) | g.lane) : 0xffffffffu);
    const int p = (int)(key >> 5), pl = (int)(key & 31u);
    const double pv = __shfl_sync(g.mask, row[k], pl, G);
    if (pv == 0.0) return k + 1;
    const double r = 1.0 / pv;
    if (g.lane == pl) {
      pos = k;
      dinv = r;
    } else if (pos == k) {
      pos = p;
    }
    const bool upd = act && pos > k;
    const double m = row[k] * r;
    if (upd) row[k] = m;
#pragma unroll
    for (int j = k + 1; j < N; ++j) {
      const double pj = __shfl_sync(g.mask, row[j], pl, G);
      if (upd) row[j] = fma(-m, pj, row[j]);
    }
  }
  return 0;
}

// the n-th set bit of m (n = 0, 1, ...), or -1
__device__ __forceinline__ int nth_bit(unsigned m, int n) {
  for (int t = 0; t < n; ++t) m &= m - 1;
  return m ? __ffs(m) - 1 : -1;
}

// ------------------------------------------------------------------ integrator
// One trip of a lane = consume the last RHS value, then run the listing
// forward until the cell needs its next RHS.  A trip is a fixed sequence of
// STAGES; every transition of the listing inside one trip goes forward in
// this order, so each lane visits each stage at most once per trip, and the
// warp reconverges (__syncwarp) between stages: lanes doing the same stage
// execute it together, whatever path brought them there.
//   CONSUME -> HIN_FINISH -> START -> SETUP(J) -> SETUP(LU) -> SOLVE -> NFAIL
//   -> ERRTEST -> STEP_TOP -> STORE -> LOAD -> ATTEMPT -> (RHS request)
// The Nordsieck vector work of a step is fused into two element-wise passes
// (registers per component): ERRTEST (complete step + the order-selection
// norms) and ATTEMPT (weights O1 + RESCALE + PREDICT + Newton start).
template <class Mech, class GM, long long SS = BDFB_TPC_BLOCK, bool MATS = true>
struct TpcIntegrator {
  static constexpr int N = Mech::N;
  using W = TWs<N, SS, MATS>;
  // warp-cooperative stages (Jacobian, LU): one cell per group of G lanes of
  // the group model GM (csrc/mech_model.cuh), GPW cells at a time per warp
  static constexpr int G = GM::G, GPW = 32 / G;
  static_assert(GM::N == N && N <= G, "group model must match the mechanism");
  static constexpr int MS = (N % 2) ? N : N + 1;                // odd smem row stride
  static constexpr int PG = N * MS + GM::SG + GM::JG;           // coop scratch doubles per group
  static constexpr int COOP_WARP = GPW * PG;
  enum : int { A_NONE = 0, A_RET, A_DONE, A_HIN_FINISH, A_START, A_SETUP, A_SETUP_J, A_SETUP_LU, A_SOLVE, A_NFAIL,
               A_ERRTEST, A_STEP_TOP, A_STORE, A_LOAD, A_ATTEMPT };
  // ATTEMPT-pass flags (TS::flag): recompute ewt from zn[0] first (O1); rescale zn[1..q] by eta^j
  // F_RESTORE: RESTORE deferred into the ATTEMPT pass (failure retries that go straight to ATTEMPT)
  // F_INCR / F_DECR: the vector part of an order change (step_top) deferred into the ATTEMPT pass; its
  // coefficients are parked in s.tq[] (rewritten by set_bdf right after that pass) and s.oc_a1
  // F_COMPLETE: cvCompleteStep (zn[j] += l_j acor, j <= qc) deferred into the ATTEMPT pass; F_FQ: zn[qmax] = acor
  // (saved for a possible order increase) deferred likewise.  Until then zn in memory is the predicted history.
  enum : int { F_EWT = 1, F_RESCALE = 2, F_RESTORE = 4, F_INCR = 8, F_DECR = 16, F_COMPLETE = 32, F_FQ = 64 };

  __device__ static double wrms_reg(const double (&v)[N], const W& w) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double p = v[i] * w.ewt(i);
      acc = acc + p * p;
    }
    return sqrt(acc / (double)N);
  }

  // RESTORE (listing): zn[j-1] -= zn[j], k = 1..q, j = q..k -- element-wise in registers
  __device__ static __noinline__ void restore(TS& s, const W& w) {
    s.tn = s.saved_t;
    const int q = s.q;
#pragma unroll 2
    for (int i = 0; i < N; ++i) {
      double z[QMAX + 1];
#pragma unroll
      for (int j = 0; j <= QMAX; ++j) z[j] = (j <= q) ? w.zn(j, i) : 0.0;
#pragma unroll
      for (int k = 1; k <= QMAX; ++k)
#pragma unroll
        for (int j = QMAX; j >= 1; --j)
          if (j >= k && j <= q) z[j - 1] = z[j - 1] - z[j];   // k <= j <= q (j >= k is compile-time)
#pragma unroll
      for (int j = 0; j < QMAX; ++j)
        if (j < q) w.zn(j, i) = z[j];
    }
  }

  // RESTORE whose vector part runs in the next ATTEMPT pass (same operations, same order)
  __device__ static void restore_deferred(TS& s) {
    s.tn = s.saved_t;
    s.flag |= F_RESTORE;
  }

  // cvSetBDF + cvSetTqBDF (scalar)
  __device__ static BDFB_HOT_INLINE void set_bdf(TS& s) {
    const int q = s.q;
    const double h = s.h;
    double xi_inv = 1.0, xistar_inv = 1.0, alpha0 = -1.0, alpha0_hat = -1.0, hsum = h;
    double* l = s.l;
    l[0] = l[1] = 1.0;
    for (int i = 2; i <= QMAX; ++i) l[i] = 0.0;
    if (q > 1) {
      for (int j = 2; j < q; ++j) {
        hsum = hsum + s.tau[j - 1];
        xi_inv = h / hsum;
        alpha0 = alpha0 - 1.0 / j;
        for (int i = j; i >= 1; --i) l[i] = l[i] + l[i - 1] * xi_inv;
      }
      alpha0 = alpha0 - 1.0 / q;
      xistar_inv = -l[1] - alpha0;
      hsum = hsum + s.tau[q - 1];
      xi_inv = h / hsum;
      alpha0_hat = -l[1] - xi_inv;
      for (int i = q; i >= 1; --i) l[i] = l[i] + l[i - 1] * xistar_inv;
    }
    const double A1 = 1.0 - alpha0_hat + alpha0;
    const double A2 = 1.0 + q * A1;
    s.tq[2] = fabs(A1 / (alpha0 * A2));
    s.tq[5] = fabs(A2 * xistar_inv / (l[q] * xi_inv));
    if (s.qwait == 1) {
      if (q > 1) {
        const double C = xistar_inv / l[q];
        const double A3 = alpha0 + 1.0 / q;
        const double A4 = alpha0_hat + xi_inv;
        const double Cpinv = (1.0 - A4 + A3) / A3;
        s.tq[1] = fabs(C * Cpinv);
      } else {
        s.tq[1] = 1.0;
      }
      hsum = hsum + s.tau[q];
      xi_inv = h / hsum;
      const double A5 = alpha0 - 1.0 / (q + 1);
      const double A6 = alpha0_hat - xi_inv;
      const double Cppinv = (1.0 - A6 + A5) / A2;
      s.tq[3] = fabs(Cppinv / (xi_inv * (q + 2) * A5));
    }
    s.tq[4] = NLSCOEF / s.tq[2];
  }

  // cvIncreaseBDF (order q -> q+1, before RESCALE: hscale = old h)
  __device__ static __noinline__ void increase_bdf(const Opts& o, TS& s, const W& w) {
    double l[QMAX + 1];
    for (int i = 0; i <= QMAX; ++i) l[i] = 0.0;
    double alpha1 = 1.0, prod = 1.0, xiold = 1.0, alpha0 = -1.0, hsum = s.hscale;
    l[2] = 1.0;
    if (s.q > 1) {
      for (int j = 1; j < s.q; ++j) {
        hsum = hsum + s.tau[j + 1];
        const double xi = hsum / s.hscale;
        prod = prod * xi;
        alpha0 = alpha0 - 1.0 / (j + 1);
        alpha1 = alpha1 + 1.0 / xi;
        for (int i = j + 2; i >= 2; --i) l[i] = l[i] * xiold + l[i - 1];
        xiold = xi;
      }
    }
    const double A1 = (-alpha0 - alpha1) / prod;
    const int q = s.q;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double zL = A1 * w.zn(o.qmax, i);
      w.zn(q + 1, i) = zL;
#pragma unroll
      for (int j = 2; j <= QMAX; ++j)
        if (j <= q) w.zn(j, i) = l[j] * zL + w.zn(j, i);
    }
  }

  // cvDecreaseBDF (order q -> q-1)
  __device__ static __noinline__ void decrease_bdf(TS& s, const W& w) {
    double l[QMAX + 1];
    for (int i = 0; i <= QMAX; ++i) l[i] = 0.0;
    l[2] = 1.0;
    double hsum = 0.0;
    for (int j = 1; j <= s.q - 2; ++j) {
      hsum = hsum + s.tau[j];
      const double xi = hsum / s.hscale;
      for (int i = j + 2; i >= 2; --i) l[i] = l[i] * xi + l[i - 1];
    }
    const int q = s.q;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double zq = w.zn(q, i);
#pragma unroll
      for (int j = 2; j < QMAX; ++j)
        if (j < q) w.zn(j, i) = -l[j] * zq + w.zn(j, i);
    }
  }

  // step_top's order change with the vector work deferred into the ATTEMPT pass (same operations, same order
  // per component; q is updated by the caller)
  __device__ static __noinline__ void order_deferred(const Opts& o, TS& s, int dq) {
    if (s.q == 2 && dq != 1) return;
    double l[QMAX + 1];
    for (int i = 0; i <= QMAX; ++i) l[i] = 0.0;
    l[2] = 1.0;
    if (dq == 1) {   // cvIncreaseBDF coefficients
      double alpha1 = 1.0, prod = 1.0, xiold = 1.0, alpha0 = -1.0, hsum = s.hscale;
      if (s.q > 1) {
        for (int j = 1; j < s.q; ++j) {
          hsum = hsum + s.tau[j + 1];
          const double xi = hsum / s.hscale;
          prod = prod * xi;
          alpha0 = alpha0 - 1.0 / (j + 1);
          alpha1 = alpha1 + 1.0 / xi;
          for (int i = j + 2; i >= 2; --i) l[i] = l[i] * xiold + l[i - 1];
          xiold = xi;
        }
      }
      s.oc_a1 = (-alpha0 - alpha1) / prod;
      s.flag |= F_INCR;
    } else {         // cvDecreaseBDF coefficients
      double hsum = 0.0;
      for (int j = 1; j <= s.q - 2; ++j) {
        hsum = hsum + s.tau[j];
        const double xi = hsum / s.hscale;
        for (int i = j + 2; i >= 2; --i) l[i] = l[i] * xi + l[i - 1];
      }
      s.flag |= F_DECR;
    }
    for (int i = 0; i <= QMAX; ++i) s.tq[i] = l[i];   // tq is free until set_bdf (prepare_next has read it)
  }

  __device__ static void adjust_order(const Opts& o, TS& s, const W& w, int dq) {
    if (s.q == 2 && dq != 1) return;
    if (dq == 1) increase_bdf(o, s, w);
    else decrease_bdf(s, w);
  }

  __device__ static void set_eta(const Opts& o, TS& s) {
    if (s.eta < THRESH) {
      s.eta = 1.0;
      s.hprime = s.h;
    } else {
      s.eta = fmin(s.eta, s.etamax);
      if (o.hmax > 0.0) s.eta = s.eta / fmax(1.0, fabs(s.h) * s.eta / o.hmax);
      s.hprime = s.h * s.eta;
    }
  }

  // RESCALE, deferred: scalar part now (h = hscale eta), zn[j] *= eta^j in the ATTEMPT pass
  __device__ static void rescale(TS& s) {
    s.flag |= F_RESCALE;
    s.rs_eta = s.eta;
    s.h = s.hscale * s.eta;
    s.hscale = s.h;
  }

  // PREPARE_NEXT (ddn = ||zn[q]||, dup = ||acor - cquot zn[qmax]||, from the complete-step pass)
  __device__ static BDFB_HOT_INLINE void prepare_next(const Opts& o, TS& s, const W& w, double dsm, double ddn,
                                                   double dup) {
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
    if (s.q > 1) etaqm1 = 1.0 / (root_l(BIAS1 * (ddn * s.tq[1]), s.q) + ADDON);
    if (s.q != o.qmax && s.saved_tq5 != 0.0) etaqp1 = 1.0 / (root_l(BIAS3 * (dup * s.tq[3]), s.L + 1) + ADDON);
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
      s.flag |= F_FQ;   // zn[qmax] = acor, in the ATTEMPT pass
    }
    set_eta(o, s);
  }

  __device__ static long long idx(const Opts& o, long long c, int k) {
    return o.layout == 0 ? (long long)k * o.ncells + c : c * (long long)N + k;
  }

  // Newton start without a predict (retry with a fresh matrix): ycor = 0, request f(tn, zn0)
  __device__ static int req_res(TS& s, const W& w) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      w.acor(i) = 0.0;
      w.yq(i) = w.zn(0, i);
    }
    s.m = 0;
    s.dprev = 0.0;
    s.tq_req = s.tn;
    s.phase = PH_NRES;
    return A_RET;
  }

  // ---- CONSUME: the RHS value fr of request s.phase is ready ------------------
  __device__ static int consume(const Opts& o, TS& s, const W& w, int rv, const double (&fr)[N]) {
    switch (s.phase) {
      case PH_NRES: {  // Newton residual: G = (rl1 zn[1] + ycor) - gamma f(tn, zn0 + ycor)
        if (rv) {
          if (s.m == 0) s.jcur = 1;   // a failed first residual is not retried (reading R5)
          return A_NFAIL;
        }
        const double rl1 = s.rl1, gm = s.gamma;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double t = rl1 * w.zn(1, i) + w.acor(i);
          w.del(i) = -gm * fr[i] + t;
        }
        return s.setup ? A_SETUP : A_SOLVE;
      }
      case PH_INIT: {  // f(t0, y0); cvHin preamble
        if (rv) { s.status = ST_RHS_FAIL; return A_STORE; }
#pragma unroll
        for (int i = 0; i < N; ++i) w.zn(1, i) = fr[i];
        if (o.h0 != 0.0) { s.hnew = o.h0; s.h = o.h0; return A_START; }
        const double tdist = o.tf - o.t0;
        const double hlb = 100.0 * (UROUND * fmax(fabs(o.t0), fabs(o.tf)));
        double hi = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double dd = HUB_FACTOR * fabs(w.zn(0, i)) + 1.0 / w.ewt(i);
          hi = fmax(hi, fabs(fr[i]) / dd);
        }
        double hub = HUB_FACTOR * tdist;
        if (hub * hi > 1.0) hub = 1.0 / hi;
        s.hub = hub;
        s.hg = sqrt(hlb * hub);
        if (hub < hlb) { s.h = s.hg; return A_START; }
        s.hs = s.hg;
        s.hnew = s.hg;
        s.count1 = 1;
        s.count2 = 1;
#pragma unroll
        for (int i = 0; i < N; ++i) w.yq(i) = s.hg * fr[i] + w.zn(0, i);
        s.tq_req = o.t0 + s.hg;
        s.phase = PH_HIN;
        return A_RET;
      }
      case PH_HIN: {  // cvYddNorm probe
        if (rv) {
          s.hg = s.hg * 0.2;
          s.count2++;
          if (s.count2 > HIN_ITERS) {
            if (s.count1 <= 2) { s.status = ST_RHS_FAIL; return A_STORE; }
            s.hnew = s.hs;
            return A_HIN_FINISH;
          }
#pragma unroll
          for (int i = 0; i < N; ++i) w.yq(i) = s.hg * w.zn(1, i) + w.zn(0, i);
          s.tq_req = o.t0 + s.hg;
          return A_RET;
        }
        const double ih = 1.0 / s.hg;
        double t[N];
#pragma unroll
        for (int i = 0; i < N; ++i) t[i] = (fr[i] - w.zn(1, i)) * ih;
        const double ydd = wrms_reg(t, w);
        s.hs = s.hg;
        s.hnew = (ydd * s.hub * s.hub > 2.0) ? sqrt(2.0 / ydd) : sqrt(s.hg * s.hub);
        if (s.count1 == HIN_ITERS) return A_HIN_FINISH;
        const double hrat = s.hnew / s.hg;
        if (hrat > 0.5 && hrat < 2.0) return A_HIN_FINISH;
        if (s.count1 > 1 && hrat > 2.0) { s.hnew = s.hg; return A_HIN_FINISH; }
        s.hg = s.hnew;
        s.count1++;
        s.count2 = 1;
#pragma unroll
        for (int i = 0; i < N; ++i) w.yq(i) = s.hg * w.zn(1, i) + w.zn(0, i);
        s.tq_req = o.t0 + s.hg;
        return A_RET;
      }
      case PH_ETF3: {  // f(tn, zn0) after the 3rd+ error-test failure at q = 1
        if (rv) { s.status = ST_RHS_FAIL; return A_STORE; }
#pragma unroll
        for (int i = 0; i < N; ++i) w.zn(1, i) = s.h * fr[i];
        return A_ATTEMPT;
      }
    }
    return A_LOAD;
  }

  __device__ static int hin_finish(const Opts& o, TS& s) {
    const double hlb = 100.0 * (UROUND * fmax(fabs(o.t0), fabs(o.tf)));
    double h = H_BIAS * s.hnew;
    if (h < hlb) h = hlb;
    if (h > s.hub) h = s.hub;
    s.h = h;
    return A_START;
  }

  __device__ static int start(const Opts& o, TS& s, const W& w) {
    double h0 = s.h;
    if (h0 > o.tf - o.t0) h0 = o.tf - o.t0;
    if (o.hmax > 0.0 && h0 > o.hmax) h0 = o.hmax;
#pragma unroll
    for (int i = 0; i < N; ++i) w.zn(1, i) = h0 * w.zn(1, i);
    s.h = s.hscale = s.hprime = h0;
    s.q = s.qprime = 1;
    s.L = 2;
    s.qwait = 2;
    s.etamax = ETAMX1;
    s.crate = 1.0;
    s.eta = 1.0;
    return A_STEP_TOP;
  }

  // cvLsSetup bookkeeping (after J and/or the factorisation)
  __device__ static void setup_done(TS& s) {
    s.nsetups++;
    s.gamrat = 1.0;
    s.gammap = s.gamma;
    s.crate = 1.0;
    s.nstlp = s.nst;
    s.setup = 0;
  }

  __device__ static int setup_decide(TS& s) {
    const double dgamma = fabs(s.gamma / s.gammap - 1.0);
    const bool jbad = (s.nst == 0) || (s.nst >= s.nstlj + MSBJ) ||
                      (s.convfail == CF_BAD_J && dgamma < DGMAX_JBAD) || (s.convfail == CF_OTHER);
    if (jbad) {
      s.nje++;
      s.nstlj = s.nst;
      s.jcur = 1;
      return A_SETUP_J;
    }
    s.jcur = 0;
    return A_SETUP_LU;
  }

  // SOLVE: delta = M^{-1}(-G), stale-gamma scaling (R6), ycor += delta, Newton test (Eq. 4)
  __device__ static int solve(TS& s, const W& w) {
    s.nni++;
    double b[N];
    tpc_solve<N, true, W::S>(&w.LU(0, 0), &w.invd(0), &w.perm(0), &w.del(0), 0, b);
    if (s.gamrat != 1.0) {
      const double sc = 2.0 / (1.0 + s.gamrat);
#pragma unroll
      for (int i = 0; i < N; ++i) b[i] = sc * b[i];
    }
    double acc = 0.0, acc2 = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double a = w.acor(i) + b[i];
      w.acor(i) = a;
      const double e = w.ewt(i);
      const double p = b[i] * e;
      acc = acc + p * p;
      const double p2 = a * e;
      acc2 = acc2 + p2 * p2;
      b[i] = a;
    }
    const double del = sqrt(acc / (double)N);
    if (s.m > 0) s.crate = fmax(CRDOWN * s.crate, del / s.dprev);
    const double dcon = del * fmin(1.0, s.crate) / s.tol;
    if (dcon <= 1.0) {
      s.acnrm = (s.m == 0) ? del : sqrt(acc2 / (double)N);
      return A_ERRTEST;
    }
    if (s.m >= 1 && del > RDIV * s.dprev) return A_NFAIL;
    s.dprev = del;
    s.m++;
    if (s.m >= MAXCOR) return A_NFAIL;
#pragma unroll
    for (int i = 0; i < N; ++i) w.yq(i) = w.zn(0, i) + b[i];
    s.tq_req = s.tn;
    s.phase = PH_NRES;
    return A_RET;
  }

  // cvHandleNFlag for a failed Newton solve
  __device__ static int nfail(const Opts& o, TS& s, const W& w) {
    if (!s.jcur) {   // retry once with a fresh Jacobian/matrix (R5)
      s.setup = 1;
      s.convfail = CF_BAD_J;
      return req_res(s, w);
    }
    s.ncfn++;
    s.ncf++;
    s.etamax = 1.0;
    if (fabs(s.h) <= o.hmin * (1.0 + UROUND) || s.ncf == MXNCF) {
      restore(s, w);
      s.status = ST_CONV_FAILURE;
      return A_STORE;
    }
    s.eta = fmax(ETACF, o.hmin / fabs(s.h));
    s.nflag = NF_PREV_CONV;
    restore_deferred(s);
    rescale(s);
    return A_ATTEMPT;
  }

  // error test; on success cvCompleteStep + PREPARE_NEXT, fused into one pass over zn
  __device__ static int errtest(const Opts& o, TS& s, const W& w) {
    const double dsm = s.acnrm * s.tq[2];
    if (dsm <= 1.0) {
      s.nst++;
      for (int i = QMAX; i >= 2; --i)
        if (i <= s.q) s.tau[i] = s.tau[i - 1];
      if (s.q == 1 && s.nst > 1) s.tau[2] = s.tau[1];
      s.tau[1] = s.h;
      s.qwait--;
      const bool fq = (s.qwait == 1 && s.q != o.qmax);
      if (fq) s.saved_tq5 = s.tq[5];
      // norms PREPARE_NEXT will need (after the complete-step update)
      const bool nn = (s.etamax != 1.0) && (s.qwait == 0);
      const bool nm1 = nn && s.q > 1;
      const bool np1 = nn && s.q != o.qmax && s.saved_tq5 != 0.0;
      double cquot = 0.0;
      if (np1) {
        const double hr = s.h / s.tau[2];
        double pw = 1.0;
        for (int k = 0; k < s.L; ++k) pw = pw * hr;
        cquot = (s.tq[5] / s.saved_tq5) * pw;
      }
      const int q = s.q, qmax = o.qmax;
      // cvCompleteStep is deferred into the next ATTEMPT pass (or STORE); here only the norms PREPARE_NEXT
      // needs, every q+1 steps: ||l_q acor + zn[q]|| and ||acor - cquot zn[qmax]|| (zn[qmax] before the
      // pass; fq and np1 are exclusive: qwait = 1 vs 0)
      s.flag |= F_COMPLETE | (fq ? F_FQ : 0);
      s.qc = q;
      double sdn = 0.0, sup = 0.0;
      if (nm1 || np1) {
        const double lq = s.l[q];
#pragma unroll kErrtestUnroll   // rounds of loads in flight
        for (int i = 0; i < N; ++i) {
          const double a = w.acor(i), e = w.ewt(i);
          if (nm1) {
            const double p = (lq * a + w.zn(q, i)) * e;
            sdn = sdn + p * p;
          }
          if (np1) {
            const double p = (-cquot * w.zn(qmax, i) + a) * e;
            sup = sup + p * p;
          }
        }
      }
      prepare_next(o, s, w, dsm, sqrt(sdn / (double)N), sqrt(sup / (double)N));
      s.etamax = ETAMX2;
      if (fabs(s.tn - o.tf) <= 100.0 * UROUND * (fabs(s.tn) + fabs(s.h))) {   // O5
        s.tn = o.tf;
        return A_STORE;
      }
      return A_STEP_TOP;
    }
    s.nef++;
    s.netf++;
    s.nflag = NF_PREV_ERR;
    if (fabs(s.h) <= o.hmin * (1.0 + UROUND) || s.nef == MXNEF) {
      restore(s, w);
      s.status = ST_ERR_FAILURE;
      return A_STORE;
    }
    s.etamax = 1.0;
    if (s.nef <= MXNEF1) {
      s.eta = 1.0 / (root_l(BIAS2 * dsm, s.L) + ADDON);
      s.eta = fmax(ETAMIN, fmax(s.eta, o.hmin / fabs(s.h)));
      if (s.nef >= SMALL_NEF) s.eta = fmin(s.eta, ETAMXF);
      restore_deferred(s);
      rescale(s);
      return A_ATTEMPT;
    }
    restore(s, w);   // the order-decrease and q = 1 paths read the restored history
    if (s.q > 1) {
      s.eta = fmax(ETAMIN, o.hmin / fabs(s.h));
      adjust_order(o, s, w, -1);
      s.L = s.q;
      s.q = s.q - 1;
      s.qwait = s.L;
      rescale(s);
      return A_ATTEMPT;
    }
    s.eta = fmax(ETAMIN, o.hmin / fabs(s.h));
    s.h = s.h * s.eta;
    s.hprime = s.h;
    s.hscale = s.h;
    s.qwait = LONG_WAIT;
#pragma unroll
    for (int i = 0; i < N; ++i) w.yq(i) = w.zn(0, i);
    s.tq_req = s.tn;
    s.phase = PH_ETF3;
    return A_RET;
  }

  // outer loop top: O1 (deferred to ATTEMPT), O2, O3, STEP prologue, order change, RESCALE
  __device__ static int step_top(const Opts& o, TS& s, const W& w) {
    if (s.nst > 0) s.flag |= F_EWT;
    if ((s.tn + s.hprime - o.tf) * s.h > 0.0) {
      s.hprime = o.tf - s.tn;
      s.eta = s.hprime / s.h;
    }
    if (s.nst >= o.mxstep) { s.status = ST_TOO_MUCH_WORK; return A_STORE; }
    s.saved_t = s.tn;
    s.ncf = 0;
    s.nef = 0;
    s.nflag = NF_FIRST;
    if (s.nst > 0 && s.hprime != s.h) {
      if (s.qprime != s.q) {
        order_deferred(o, s, s.qprime - s.q);
        s.q = s.qprime;
        s.L = s.q + 1;
        s.qwait = s.L;
      }
      rescale(s);
    }
    return A_ATTEMPT;
  }

  // ATTEMPT: one pass over zn -- [ewt (O1)] [RESCALE] PREDICT, ycor = 0, yq = zn0; then SET_BDF etc.
  __device__ static int attempt(const Opts& o, TS& s, const W& w, const double* atol) {
    const int fl = s.flag;
    s.flag = 0;
    const int q = s.q;
    double f[QMAX + 1];
    f[0] = 1.0;
    {
      const double eta = (fl & F_RESCALE) ? s.rs_eta : 1.0;
      double g = eta;
#pragma unroll
      for (int j = 1; j <= QMAX; ++j) {
        f[j] = g;
        g = g * eta;
      }
    }
    const double rtol = o.rtol;
    constexpr int CH = BDFB_ATTEMPT_CH ? BDFB_ATTEMPT_CH : ((N % 4 == 0) ? 4 : 2);   // elements per chunk
    static_assert(N % CH == 0, "chunking");
    // rows to read: the new order, the old zn[q + 1] of a deferred decrease, the rows of a deferred completion
    const int qc = (fl & F_COMPLETE) ? s.qc : 0;
    const int qdec = q + ((fl & F_DECR) ? 1 : 0);
    const int qld = qdec > qc ? qdec : qc;
    const int qwb = q > qc ? q : qc;                  // rows written back (a completed row above a decrease)
    double lk[QMAX + 1], lc[QMAX + 1];
#pragma unroll
    for (int j = 0; j <= QMAX; ++j) {
      lk[j] = s.l[j];    // step coefficients of the deferred completion
      lc[j] = s.tq[j];   // order-change coefficients (order_deferred)
    }
    const double a1 = s.oc_a1;
    const int qmx = o.qmax;
    const bool wqmax = (fl & F_FQ) && qmx > qwb;      // zn[qmax] = acor lands in its own row
#pragma unroll kAttemptUnroll
    for (int i0 = 0; i0 < N; i0 += CH) {
      double zc[CH][QMAX + 1], zm[CH], ac[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
#pragma unroll
        for (int j = 0; j <= QMAX; ++j) zc[c][j] = (j <= qld) ? w.zn(j, i0 + c) : 0.0;
        ac[c] = (fl & F_COMPLETE) ? w.acor(i0 + c) : 0.0;
        zm[c] = ((fl & F_INCR) && !(fl & F_FQ)) ? w.zn(qmx, i0 + c) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int i = i0 + c;
        double* z = zc[c];
        if (fl & F_COMPLETE) {   // deferred cvCompleteStep: zn[j] = l_j acor + zn[j], j <= qc
#pragma unroll
          for (int j = 0; j <= QMAX; ++j)
            if (j <= qc) z[j] = lk[j] * ac[c] + z[j];
          if (fl & F_FQ) zm[c] = ac[c];               // zn[qmax] = acor (read by an order increase)
        }
        if (fl & F_RESTORE) {   // deferred RESTORE (q unchanged since the failed attempt)
#pragma unroll
          for (int k = 1; k <= QMAX; ++k)
#pragma unroll
            for (int j = QMAX; j >= 1; --j)
              if (j >= k && j <= q) z[j - 1] = z[j - 1] - z[j];
        }
        if (fl & F_INCR) {   // cvIncreaseBDF, vector part (q = old q + 1): zn[q] = A1 zn[qmax], zn[j] += l_j zn[q]
          const double zL = a1 * zm[c];
#pragma unroll
          for (int j = 2; j < QMAX; ++j)
            if (j < q) z[j] = lc[j] * zL + z[j];
#pragma unroll
          for (int j = 2; j <= QMAX; ++j)
            if (j == q) z[j] = zL;
        }
        if (fl & F_DECR) {   // cvDecreaseBDF, vector part (q = old q - 1): zn[j] -= l_j zn[old q]
          double zq = 0.0;
#pragma unroll
          for (int j = 2; j <= QMAX; ++j)
            if (j == q + 1) zq = z[j];
#pragma unroll
          for (int j = 2; j < QMAX; ++j)
            if (j <= q) z[j] = -lc[j] * zq + z[j];
        }
        if (fl & F_EWT) w.ewt(i) = 1.0 / (rtol * fabs(z[0]) + atol[i]);
        if (fl & F_RESCALE) {
#pragma unroll
          for (int j = 1; j <= QMAX; ++j)
            if (j <= q) z[j] = f[j] * z[j];
        }
#pragma unroll
        for (int k = 1; k <= QMAX; ++k)
#pragma unroll
          for (int j = QMAX; j >= 1; --j)
            if (j >= k && j <= q) z[j - 1] = z[j - 1] + z[j];
#pragma unroll
        for (int j = 0; j <= QMAX; ++j)
          if (j <= qwb) w.zn(j, i) = z[j];
        if (wqmax) w.zn(qmx, i) = ac[c];
        w.yq(i) = z[0];
        w.acor(i) = 0.0;
      }
    }
    s.tn = s.tn + s.h;
    if ((s.tn - o.tf) * s.h > 0.0) s.tn = o.tf;
    set_bdf(s);
    s.rl1 = 1.0 / s.l[1];
    s.gamma = s.h * s.rl1;
    if (s.nst == 0) s.gammap = s.gamma;
    s.gamrat = (s.nst > 0) ? s.gamma / s.gammap : 1.0;
    s.convfail = (s.nflag == NF_FIRST || s.nflag == NF_PREV_ERR) ? CF_NONE : CF_OTHER;
    s.setup = (s.nflag == NF_PREV_CONV) || (s.nflag == NF_PREV_ERR) || (s.nst == 0) ||
              (s.nst >= s.nstlp + MSBP) || (fabs(s.gamrat - 1.0) > DGMAX);
    s.tol = s.tq[4];
    s.jcur = 0;
    s.m = 0;
    s.dprev = 0.0;
    s.tq_req = s.tn;
    s.phase = PH_NRES;
    return A_RET;
  }

  __device__ static void store(const Opts& o, TS& s, const W& w, double* y, Agg& acc, const CellStatsPtrs& cs) {
    const long long c = s.cell;
    if (s.status != ST_NONFINITE) {
      const bool pend = (s.flag & F_COMPLETE) != 0;   // the last step's completion is still deferred
      const double l0 = s.l[0];
#pragma unroll
      for (int i = 0; i < N; ++i) y[idx(o, c, i)] = pend ? l0 * w.acor(i) + w.zn(0, i) : w.zn(0, i);
    }
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
    atomicAdd(&acc.n_failed, (unsigned long long)(s.status != ST_OK));
    atomicAdd(&acc.nst, (unsigned long long)s.nst);
    atomicAdd(&acc.nfe, (unsigned long long)s.nfe);
    atomicAdd(&acc.nje, (unsigned long long)s.nje);
    atomicAdd(&acc.nsetups, (unsigned long long)s.nsetups);
    atomicAdd(&acc.nni, (unsigned long long)s.nni);
    atomicAdd(&acc.netf, (unsigned long long)s.netf);
    atomicAdd(&acc.ncfn, (unsigned long long)s.ncfn);
    atomicMax(&acc.nst_max, (unsigned long long)s.nst);
    atomicMax(&acc.nfe_max, (unsigned long long)s.nfe);
    atomicAdd(&acc.cells_done, 1ull);
  }

  // next cell from the device work counter: A_RET (f(t0, y0) requested) or A_DONE
  __device__ static int load(const Opts& o, TS& s, const W& w, double* y, const double* fext, const double* aux,
                             const double* atol, unsigned long long* counter, Agg& acc, const CellStatsPtrs& cs) {
    for (;;) {
      const long long c = (long long)atomicAdd(counter, 1ull);
      if (c >= o.ncells) { s.phase = PH_DONE; return A_DONE; }
      s.cell = c;
      s.aux = aux ? aux[c] : 0.0;
      int bad = !isfinite(s.aux);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double y0 = y[idx(o, c, i)];
        const double fe = fext ? fext[idx(o, c, i)] : 0.0;
        if (!isfinite(y0) || !isfinite(fe)) bad = 1;
        w.zn(0, i) = y0;
        w.fext(i) = fe;
        w.acor(i) = 0.0;
        w.yq(i) = y0;
        w.ewt(i) = 1.0 / (o.rtol * fabs(y0) + atol[i]);
      }
      for (int j = 1; j <= QMAX; ++j) {
#pragma unroll
        for (int i = 0; i < N; ++i) w.zn(j, i) = 0.0;
      }
      s.nst = s.nfe = s.nje = s.nsetups = s.nni = s.netf = s.ncfn = 0;
      s.nstlp = s.nstlj = 0;
      s.status = ST_OK;
      s.tn = o.t0;
      s.q = 1;
      s.h = 0.0;
      for (int i = 0; i <= QMAX + 1; ++i) s.tau[i] = 0.0;
      for (int i = 0; i <= QMAX; ++i) s.l[i] = 0.0;
      for (int i = 0; i < 6; ++i) s.tq[i] = 0.0;
      s.saved_tq5 = 0.0;
      s.gammap = 0.0;
      s.gamrat = 1.0;
      s.acnrm = 0.0;
      s.crate = 1.0;
      s.flag = 0;
      if (bad) {
        s.status = ST_NONFINITE;
        store(o, s, w, y, acc, cs);
        continue;
      }
      s.tq_req = o.t0;
      s.phase = PH_INIT;
      return A_RET;
    }
  }

  // one trip (all lanes of the warp call it; dead lanes only take part in the syncs)
  // scalar state / workspace of lane l of this warp
  __device__ static TS& ts_of(int l) {
    extern __shared__ double smem[];
    return *reinterpret_cast<TS*>(smem + ((threadIdx.x & ~31u) + l) * TS_STRIDE);
  }
  __device__ static W ws_of(int l);
  // block-packed LU list: BLOCK thread ids + per-warp counts (ints, after the coop scratch)
  __device__ static int* lu_list() {
    extern __shared__ double smem[];
    return reinterpret_cast<int*>(smem + BDFB_TPC_BLOCK * TS_STRIDE + 2 + (BDFB_TPC_BLOCK / 32) * (sizeof(Agg) / 8) +
                                  (size_t)(BDFB_TPC_BLOCK / 32) * COOP_WARP);
  }

  __device__ static int trip(const Opts& o, TS& s, const W& w, bool live, int rv, const double (&fr)[N], double* y,
                             const double* fext, const double* aux, const double* atol, unsigned long long* counter,
                             Agg& acc, const CellStatsPtrs& cs, double* coop) {
    int act = live ? consume(o, s, w, rv, fr) : A_DONE;
    if (act == A_HIN_FINISH) act = hin_finish(o, s);
    if (act == A_START) act = start(o, s, w);
    if (act == A_SETUP) act = setup_decide(s);
    __syncwarp();
    // ---- SETUP (J): warp-cooperative, one cell per group of G lanes, over the
    // lanes that need a fresh Jacobian (table-driven group code of mech_model.cuh)
    const int gi = (int)(threadIdx.x & 31) / G;
    {
      Grp<G> g;
      double* cs_g = coop + gi * PG;            // [J rows (stride MS) | SG | JG]
      unsigned mask = __ballot_sync(0xffffffffu, act == A_SETUP_J);
      while (mask) {
        const int l = nth_bit(mask, gi);
        for (int t = 0; t < GPW; ++t) mask &= mask - 1;
        if (l >= 0) {
          TS& sl = ts_of(l);
          const W wl = ws_of(l);
          const double yv = g.lane < N ? wl.yq(g.lane) : 0.0;
          const int r = GM::template jac<MS>(g, yv, sl.aux, cs_g + g.lane, cs_g + N * MS, cs_g + N * MS + GM::SG);
          if (!r && g.lane < N) {
#pragma unroll 2
            for (int j = 0; j < N; ++j) wl.J(g.lane, j) = cs_g[j * MS + g.lane];
          }
          if (g.lane == 0) sl.coop = r;
        }
        __syncwarp();
      }
    }
    if (act == A_SETUP_J) {
      if (s.coop) {
        setup_done(s);
        act = A_NFAIL;
      } else {
        act = A_SETUP_LU;
      }
    }
    __syncwarp();
#if BDFB_TPC_LU == 0
    // ---- SETUP (LU), block-packed: the block's cells that need a factorisation
    // this trip (about 19% of them) are compacted in thread order into a list,
    // and warps take 32 list entries at a time -- every lane factors one cell
    // (M = I - gamma J fused into the left-looking LU), so the O(n^3) work runs
    // on full warps instead of on the ~6 lanes per warp that need it.
    {
      int* lst = lu_list();
      const unsigned ball = __ballot_sync(0xffffffffu, act == A_SETUP_LU);
      const int lane = (int)(threadIdx.x & 31), warp = (int)(threadIdx.x >> 5);
      if (lane == 0) lst[BDFB_TPC_BLOCK + warp] = __popc(ball);
      __syncthreads();
      int off = 0, tot = 0;
#pragma unroll
      for (int v = 0; v < BDFB_TPC_BLOCK / 32; ++v) {
        const int c = lst[BDFB_TPC_BLOCK + v];
        off += (v < warp) ? c : 0;
        tot += c;
      }
      if (act == A_SETUP_LU) lst[off + __popc(ball & ((1u << lane) - 1u))] = (int)threadIdx.x;
      __syncthreads();
      for (int it = warp * 32 + lane; it - lane < tot; it += BDFB_TPC_BLOCK) {
        if (it < tot) {
          const int t = lst[it];
          const W wt = ws_of(t - (int)(threadIdx.x & ~31u));
          TS& st = ts_of(t - (int)(threadIdx.x & ~31u));
          st.coop = tpc_factor<N, true, W::S>(&wt.J(0, 0), &wt.LU(0, 0), &wt.invd(0), &wt.perm(0), 0, st.gamma,
                                              nullptr);
        }
      }
      __syncthreads();
    }
#elif BDFB_TPC_LU == 2
    // ---- SETUP (LU): M = I - gamma J fused into the per-lane left-looking LU (lanes in place)
    if (act == A_SETUP_LU) {
      const int r = tpc_factor<N, true, W::S>(&w.J(0, 0), &w.LU(0, 0), &w.invd(0), &w.perm(0), 0, s.gamma, nullptr);
      s.coop = r;
    }
#else
    // ---- SETUP (LU): M = I - gamma J, warp-cooperative factorisation
    {
      Grp<G> g;
      unsigned mask = __ballot_sync(0xffffffffu, act == A_SETUP_LU);
      while (mask) {
        const int l = nth_bit(mask, gi);
        for (int t = 0; t < GPW; ++t) mask &= mask - 1;
        if (l >= 0) {
          TS& sl = ts_of(l);
          const W wl = ws_of(l);
          const double gm = sl.gamma;
          const int i = g.lane;
          double row[N];
#pragma unroll
          for (int j = 0; j < N; ++j) row[j] = (i < N) ? (i == j ? 1.0 : 0.0) - gm * wl.J(i, j) : 0.0;
          int pos;
          double dinv;
          const int r = coop_factor<N, G>(g, row, pos, dinv);
          if (!r && i < N) {
#pragma unroll
            for (int j = 0; j < N; ++j) wl.LU(pos, j) = row[j];
            wl.perm(pos) = i;
            wl.invd(pos) = dinv;
          }
          if (g.lane == 0) sl.coop = r;
        }
        __syncwarp();
      }
    }
#endif
    if (act == A_SETUP_LU) {
      setup_done(s);
      act = s.coop ? A_NFAIL : A_SOLVE;
    }
    __syncwarp();
    if (act == A_SOLVE) act = solve(s, w);
    __syncwarp();
    if (act == A_NFAIL) act = nfail(o, s, w);
    __syncwarp();
    if (act == A_ERRTEST) act = errtest(o, s, w);
    __syncwarp();
    if (act == A_STEP_TOP) act = step_top(o, s, w);
    __syncwarp();
    if (act == A_STORE) {
      store(o, s, w, y, acc, cs);
      act = A_LOAD;
    }
    if (act == A_LOAD) act = load(o, s, w, y, fext, aux, atol, counter, acc, cs);
    __syncwarp();
    if (act == A_ATTEMPT) act = attempt(o, s, w, atol);
    __syncwarp();
    return act;
  }
};

template <class Mech, class GM, long long SS, bool MATS>
__device__ typename TpcIntegrator<Mech, GM, SS, MATS>::W TpcIntegrator<Mech, GM, SS, MATS>::ws_of(int l) {
  extern __shared__ double smem[];
  double* const* bases = reinterpret_cast<double* const*>(smem + BDFB_TPC_BLOCK * TS_STRIDE);
  int* const* ibases = reinterpret_cast<int* const*>(smem + BDFB_TPC_BLOCK * TS_STRIDE + 1);
  const int t = (int)(threadIdx.x & ~31u) + l;
  return W{bases[0] + t, ibases[0] + t};
}

// shared memory: [TS x BLOCK][ws base, iws base][Agg x warps][coop scratch x warps]
template <class Mech, class GM>
constexpr size_t tpc_smem_bytes() {
  using I = TpcIntegrator<Mech, GM>;
  return sizeof(double) * ((size_t)BDFB_TPC_BLOCK * TS_STRIDE + 2 + (BDFB_TPC_BLOCK / 32) * (sizeof(Agg) / 8) +
                           (size_t)(BDFB_TPC_BLOCK / 32) * I::COOP_WARP) +
         sizeof(int) * (BDFB_TPC_BLOCK + BDFB_TPC_BLOCK / 32);
}

template <class Mech, class GM>
__global__ void __launch_bounds__(BDFB_TPC_BLOCK, BDFB_TPC_MINB)
    integrate_tpc_kernel(Opts o, double* y, const double* fext, const double* aux, const double* atol, double* ws,
                         int* iws, unsigned long long* counter, Agg* agg, CellStatsPtrs cs) {
  using I = TpcIntegrator<Mech, GM>;
  constexpr int N = Mech::N;
  extern __shared__ double smem[];
  __shared__ double satol[N];
  if (threadIdx.x < N) satol[threadIdx.x] = atol[threadIdx.x];
  const int warp = threadIdx.x >> 5;
  TS& s = *reinterpret_cast<TS*>(smem + threadIdx.x * TS_STRIDE);
  double* bases = smem + BDFB_TPC_BLOCK * TS_STRIDE;
  Agg& acc = *reinterpret_cast<Agg*>(bases + 2 + warp * (sizeof(Agg) / 8));
  double* coop = bases + 2 + (BDFB_TPC_BLOCK / 32) * (sizeof(Agg) / 8) + warp * I::COOP_WARP;
  double* wsb = ws + (long long)blockIdx.x * TWs<N>::DOUBLES * BDFB_TPC_BLOCK;
  int* iwsb = iws + (long long)blockIdx.x * TWs<N>::INTS * BDFB_TPC_BLOCK;
  if (threadIdx.x == 0) {
    reinterpret_cast<double**>(bases)[0] = wsb;
    reinterpret_cast<int**>(bases + 1)[0] = iwsb;
  }
  if ((threadIdx.x & 31) == 0) acc = Agg{};
  const TWs<N> w{wsb + threadIdx.x, iwsb + threadIdx.x};
  s.phase = PH_DONE;
  s.flag = 0;
  __syncthreads();
  int rv = 0;
  double fr[N];
#pragma unroll
  for (int i = 0; i < N; ++i) fr[i] = 0.0;
  bool live = true;
  for (;;) {
    live = I::trip(o, s, w, live, rv, fr, y, fext, aux, satol, counter, acc, cs, coop) == I::A_RET;
#ifndef BDFB_NO_BLOCK_SYNC
    __syncwarp();   // reconverge the warp before the block barrier (synccheck)
    if (!__syncthreads_or(live)) break;
#else
    if (!__any_sync(0xffffffffu, live)) break;
#endif
    if (live) {
      double yv[N];
#pragma unroll
      for (int i = 0; i < N; ++i) yv[i] = w.yq(i);
      rv = Mech::rhs(yv, s.aux, fr);
#pragma unroll
      for (int i = 0; i < N; ++i) fr[i] = fr[i] + w.fext(i);
      s.nfe++;
    }
  }
  // aggregate statistics: the warp's shared accumulators, one atomic per counter per warp
  __syncwarp();
  if ((threadIdx.x & 31) == 0 && acc.cells_done) {
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
