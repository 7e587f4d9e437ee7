// bdf_split.cuh -- the SPLIT organisation of the per-cell BDF integrator for
// the reacting-flow mechanism models (B200 / sm_100a).
//
// Semantics: the listing SURVEY.md §8(c).2 (CVODE's fixed-leading-coefficient
// Nordsieck BDF), executed by the same
// thread-per-cell state machine as bdf_tpc.cuh (TpcIntegrator: one cell per
// lane, identical stages, constants and operation order; WRMS order R15 with
// G = 1; LU bit-identical to LU_FACTOR, reading R16).
//
// Why split (ncu, profiles/r1): one persistent kernel that holds a cell's
// whole life -- RHS, Jacobian, LU and control -- keeps only 8 warps per SM
// resident (its straight-line RHS needs 255 registers), serialises the
// block's LU work onto one warp behind __syncthreads (barrier stalls), and
// re-reads every L entry of its factorisations from L2/HBM (long-scoreboard
// stalls): FP64 pipe < 5%, IPC 0.27.  Here a pool of S cell SLOTS lives in
// HBM between launches and every trip of the listing runs as five kernels,
// each with its own register budget, occupancy and memory pattern:
//
//   K_ctl (pass A, thread per slot, all slots): consume the RHS value;
//     cvHin; decide the matrix setup.  A cell that needs no setup continues
//     (Newton solve with its LU, error test, step/order selection, order
//     change, predictor) to its next RHS request; one that needs a setup
//     stops and joins the setup list (and the Jacobian list if J is stale).
//     A finished cell is stored and the slot loads the next cell from the
//     device work counter, so the pool stays full until the counter runs out
//     (per-cell adaptive stepping: a stiff cell holds its slot for more trips).
//   K_jac (Jacobian list): the generated analytic Jacobian in two passes --
//     reactions in warp-uniform parts + an ordered sum (thread per cell and
//     part), then one column per thread -- into the slot's J record.
//   K_lu (setup list, one cell per group of 8 lanes, 4 per warp): M = I - gamma J,
//     LU with partial pivoting in registers (oct_factor), factors stored
//     column-major in pivoted row order with 1/U_kk and the permutation.
//   K_ctl (pass B, thread per listed slot): the rest of the trip after the
//     setup, to the next RHS request.
//   K_rhs (thread per slot with a request): f = R(yq) + F, generated
//     straight-line RHS -- the transcendental-heavy FP64 work on full warps.
//
// HBM records per slot s (all allocated once, sized for the pool):
//   VEC  warp-blocked SoA: element e of slot s at vec[((s/32) D + e) 32 + s%32]
//        (zn[0..5], ewt, acor, yq, del, fext, 1/U_kk (unused), fr): a warp of
//        consecutive slots reads one element as one 256-byte line;
//   TS   the scalar state (struct TS), one record per slot, block-contiguous
//        (K_ctl copies its block's records through shared memory);
//   J    column-major n x n (LUREC stride);
//   LU   column-major n x n factors in pivoted row order | 1/U_kk[n] | perm[n]
//        (ints): the Newton solve of a thread streams its own record with
//        16-byte loads, column by column in the order of the substitutions.
#pragma once
#include <utility>

#include "bdf_tpc.cuh"

namespace bdfb {

#ifndef BDFB_SPLIT_BLOCK
#define BDFB_SPLIT_BLOCK 128
#endif
// K_ctl block size (a block retires when its slowest warp finishes: small blocks waste less)
#ifndef BDFB_SPLIT_CTL_BLOCK
#define BDFB_SPLIT_CTL_BLOCK 128
#endif
#ifndef BDFB_SPLIT_CTL_MINB
#define BDFB_SPLIT_CTL_MINB 3
#endif
// 1: K_ctl stages each warp's TS records through shared memory; 0: accesses them in HBM (L1-cached)
#ifndef BDFB_SPLIT_TS_SMEM
#define BDFB_SPLIT_TS_SMEM 1
#endif
#ifndef BDFB_SPLIT_PREFETCH
#define BDFB_SPLIT_PREFETCH 0
#endif
// 1: cell start/end (store, load, cvHin) in a separate compacted kernel K_init (full warps of starting cells)
#ifndef BDFB_SPLIT_INIT_KERNEL
#define BDFB_SPLIT_INIT_KERNEL 0   // measured slower on C4 (K_ctl+K_init 3.80 s vs K_ctl 3.34 s): kept as an option
#endif

// split-local phases: waiting for the setup kernels; finished, to be stored by K_init; a Jv request of GMRES
constexpr int PH_SETUP = 6, PH_STORE = 7, PH_KRY = 8;

// 1: K_rhs also runs the Newton residual and the LU solve of a PH_NRES request whose matrix is current (dense
// direct solver, n <= 32), so that the 4 KB LU-record stream of the solve leaves the memory-bound, divergent
// K_ctl; K_ctl then finds the correction in the del row (rv = RV_SOLVED) and runs only the Newton update and
// test (same operations, same order).  Measured on C4: K_ctl 3274 -> 3155 ms but K_rhs 933 -> 2560 ms (the
// stream stalls the RHS warps instead of overlapping them): off, kept as an option.
#ifndef BDFB_SPLIT_RHS_SOLVE
#define BDFB_SPLIT_RHS_SOLVE 0
#endif
constexpr int RV_SOLVED = -1;   // b.rv code: K_rhs returned f = R + F consumed and delta = M^-1 (-G) in del

// linear solver inside the Newton iteration (bdfb_set_linear_solver; Table 1)
enum : int { LS_DENSE = 0, LS_DIAG = 1, LS_GMRES = 2 };
constexpr int KMAXL = 5;            // Krylov dimension of the VEC record (CVODE's default maxl; reading R29)
constexpr double EPLIFAC = 0.05;    // c_l of Eq. 6
constexpr int MAX_DQITERS = 3;      // Jv difference quotient: tries with sigma /= 4 after an RHS failure

struct SplitBufs {
  double* vec;                 // S/32 * D * 32
  double* ts;                  // S * TS_STRIDE
  double* J;                   // S * JREC
  double* LU;                  // S * LUREC
  double* jscr;                // two-pass Jacobian scratch, Jacobian-list entry e, element r at
                               // jscr[((e/32) NSC2 + r) 32 + e%32] (S * NSC2; null when unused)
  int* rv;                     // S: RHS status of the last request
  int* slist;                  // setup list (slots)
  int* jlist;                  // Jacobian list (slots)
  int* ilist;                  // cell start/end list (slots for K_init)
  unsigned* cnt;               // [3 (it & 1) + {0, 1, 2}]: setup, Jacobian, K_init list counts of iteration it
  unsigned long long* live;    // [2]: live slots after the K_ctl of iteration it (it & 1)
  long long slots;             // S (multiple of 32)
  int jac_dq;                  // 1: difference-quotient Jacobian (K_dqjac) instead of the analytic one
  int maxl;                    // LS_GMRES: Krylov iterations per linear solve, 1..KMAXL
};

// LU record layout: 1 = each slot's record contiguous (a thread streams its own record with 16-byte loads;
// every warp load touches 32 lines); 32 = warp-blocked SoA like VEC, element e of slot s at
// LU[((s/32) LUREC + e) 32 + s%32] (a warp load of one element is one coalesced 256-byte access)
#ifndef BDFB_SPLIT_LU_SOA
#define BDFB_SPLIT_LU_SOA 0   // measured on C4: K_ctl -4% but K_lu 1.05 -> 2.22 s (scattered 8-byte writes): off
#endif
constexpr int LU_STRIDE = BDFB_SPLIT_LU_SOA ? 32 : 1;

// VEC layout: 0 = warp-blocked SoA (element e of slot s at vec[((s/32) D + e) 32 + s%32]: a warp of consecutive
// slots reads one element as one 256-byte line); 1 = slot-major (slot s's D doubles contiguous: a lane's rows are
// its own lines, so lanes that sit out a divergent stage fetch no sectors)
#ifndef BDFB_SPLIT_VEC_AOS
#define BDFB_SPLIT_VEC_AOS 0
#endif
constexpr int VEC_S = BDFB_SPLIT_VEC_AOS ? 1 : 32;

// Substitutions of LU_SOLVE (listing; reading R16) on a column-major LU
// record (factors in pivoted row order | 1/U_kk | perm), b already permuted:
// unit-L forward substitution column by column, then the back substitution
// with the reciprocal diagonal -- the operations and order of the oracle's
// orc_lu_solve.  Shared by the Newton solve of K_ctl and the LU diagnostic.
// S: element stride of the record (LU_STRIDE).
template <int N, int S>
__device__ __forceinline__ void lurec_substitute(const double* __restrict__ lu, double (&b)[N]) {
  constexpr int LU_INVD = N * N;
  if constexpr (S != 1) {
#pragma unroll
    for (int k = 0; k < N - 1; ++k) {         // unit-L forward substitution, column k
#pragma unroll
      for (int i = k + 1; i < N; ++i) b[i] = fma(-lu[(k * N + i) * S], b[k], b[i]);
    }
    double inv[N];
#pragma unroll
    for (int i = 0; i < N; ++i) inv[i] = lu[(LU_INVD + i) * S];
#pragma unroll
    for (int k = N - 1; k > 0; --k) {         // back substitution, column k, reciprocal diagonal
      b[k] = b[k] * inv[k];
#pragma unroll
      for (int i = 0; i < k; ++i) b[i] = fma(-lu[(k * N + i) * S], b[k], b[i]);
    }
    b[0] = b[0] * inv[0];
    return;
  }
  const double2* col = reinterpret_cast<const double2*>(lu);
#pragma unroll
  for (int k = 0; k < N - 1; ++k) {           // unit-L forward substitution, column k
    double c[N];
#pragma unroll
    for (int h = (k + 1) / 2; h < N / 2; ++h) {
      const double2 v = col[(k * N) / 2 + h];
      c[2 * h] = v.x;
      c[2 * h + 1] = v.y;
    }
#pragma unroll
    for (int i = k + 1; i < N; ++i) b[i] = fma(-c[i], b[k], b[i]);
  }
  const double2* inv2 = reinterpret_cast<const double2*>(lu + LU_INVD);
  double inv[N];
#pragma unroll
  for (int h = 0; h < N / 2; ++h) {
    const double2 v = inv2[h];
    inv[2 * h] = v.x;
    inv[2 * h + 1] = v.y;
  }
#pragma unroll
  for (int k = N - 1; k > 0; --k) {           // back substitution, column k, reciprocal diagonal
    b[k] = b[k] * inv[k];
    double c[N];
#pragma unroll
    for (int h = 0; h < (k + 1) / 2; ++h) {
      const double2 v = col[(k * N) / 2 + h];
      c[2 * h] = v.x;
      c[2 * h + 1] = v.y;
    }
#pragma unroll
    for (int i = 0; i < k; ++i) b[i] = fma(-c[i], b[k], b[i]);
  }
  b[0] = b[0] * inv[0];
}

template <class Mech, class GM, int LS = LS_DENSE>
struct Split {
  static constexpr int N = Mech::N;
  using I = TpcIntegrator<Mech, GM, VEC_S, false>;
  using W = typename I::W;
  static constexpr int D0 = W::DOUBLES;
  // extra VEC elements of the matrix-free linear solvers.  CVDiag: f at the setup point, gamma of the
  // diagonal (M^-1 itself lives in W::invd).  GMRES: Krylov basis V[0..KMAXL] (scaled), fy = f(ycur), the
  // rotated Hessenberg matrix H[KMAXL+1][KMAXL], Givens pairs, sigma, beta, rotation product, l, Jv retries,
  // linear iterations of the cell.
  static constexpr int X_FT = D0, X_GSV = D0 + N;
  static constexpr int X_V = D0, X_FY = X_V + (KMAXL + 1) * N, X_H = X_FY + N, X_GIV = X_H + (KMAXL + 1) * KMAXL,
                       X_SIG = X_GIV + 2 * KMAXL, X_BETA = X_SIG + 1, X_ROT = X_BETA + 1, X_L = X_ROT + 1,
                       X_DQ = X_L + 1, X_NLI = X_DQ + 1, X_END = X_NLI + 1;
  static constexpr int D = (LS == LS_DENSE || LS == 3 /* LS_ERK: erk_split.cuh */)
                               ? D0 : (LS == LS_DIAG ? ((D0 + N + 1 + 1) & ~1) : ((X_END + 1) & ~1));
  static constexpr int JREC = (N * N + 3) / 4 * 4;
  static constexpr int LU_INVD = N * N, LU_PERM = N * N + N;     // perm: ints at double offset LU_PERM
  // perm: ints at double offset LU_PERM (contiguous records) or one double element per entry (SoA)
  static constexpr int LUREC = LU_STRIDE == 1 ? (N * N + N + (N + 1) / 2 + 3) / 4 * 4 : N * N + 2 * N;
  __device__ static double* lurec(const SplitBufs& b, long long slot) {
    return LU_STRIDE == 1 ? b.LU + slot * LUREC : b.LU + ((slot >> 5) * LUREC) * 32 + (slot & 31);
  }
  __device__ static int lu_perm(const double* lu, int i) {
    if constexpr (LU_STRIDE == 1) return reinterpret_cast<const int*>(lu + LU_PERM)[i];
    else return (int)lu[(LU_PERM + i) * LU_STRIDE];
  }
  static_assert(N % 2 == 0, "16-byte column loads need an even n");
  static_assert(sizeof(TS) <= sizeof(double) * TS_STRIDE, "TS record");

  __device__ static W ws(const SplitBufs& b, long long slot) {
    if constexpr (VEC_S == 1) return W{b.vec + slot * D, nullptr};
    else return W{b.vec + ((slot >> 5) * D) * 32 + (slot & 31), nullptr};
  }
  __device__ static TS* ts(const SplitBufs& b, long long slot) {
    return reinterpret_cast<TS*>(b.ts + slot * TS_STRIDE);
  }

  // SOLVE with the slot's LU record (listing LU_SOLVE, reading R16): the
  // same operations in the same order as tpc_solve, then the stale-gamma
  // scaling, ycor update and the Newton test of TpcIntegrator::solve.
  __device__ static int solve(TS& s, const W& w, const double* __restrict__ lu) {
    s.nni++;
    double b[N];
#pragma unroll
    for (int i = 0; i < N; ++i) b[i] = -w.del(lu_perm(lu, i));
    lurec_substitute<N, LU_STRIDE>(lu, b);
    if (s.gamrat != 1.0) {
      const double sc = 2.0 / (1.0 + s.gamrat);
#pragma unroll
      for (int i = 0; i < N; ++i) b[i] = sc * b[i];
    }
    return newton_update(s, w, b);
  }

  // the Newton residual and the substitutions already ran in K_rhs (RV_SOLVED): delta is in the del row
  __device__ static int solved(TS& s, const W& w) {
    s.nni++;
    double x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = w.del(i);
    return newton_update(s, w, x);
  }

  // ycor += delta, ||delta|| and the Newton test of Eq. 4 (TpcIntegrator::solve's tail), for every linear solver
  __device__ static int newton_update(TS& s, const W& w, double (&b)[N]) {
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
      return I::A_ERRTEST;
    }
    if (s.m >= 1 && del > RDIV * s.dprev) return I::A_NFAIL;
    s.dprev = del;
    s.m++;
    if (s.m >= MAXCOR) return I::A_NFAIL;
#pragma unroll
    for (int i = 0; i < N; ++i) w.yq(i) = w.zn(0, i) + b[i];
    s.tq_req = s.tn;
    s.phase = PH_NRES;
    return I::A_RET;
  }

  // ---- CVDiag (LS_DIAG, listing "Variant for n=1 / C2" for any n; oracle lsetup/lsolve) ----------
  // setup part 1 (at the matrix-setup decision; fr = f(y) of the residual just consumed): the perturbed
  // state y + r (h f - zn[1]), r = FRACT rl1, is requested from K_rhs
  __device__ static int diag_request(TS& s, const W& w) {
    const double r = FRACT * s.rl1;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double ft0 = w.fr(i);
      w.at(X_FT + i) = ft0;
      const double ft = s.h * ft0 - w.zn(1, i);
      w.yq(i) = r * ft + w.yq(i);
    }
    s.nje++;
    s.jcur = 1;
    s.tq_req = s.tn;
    s.phase = PH_DIAG;
    return I::A_RET;
  }
  // setup part 2: M_ii = (FRACT ft + (-h)(f(yp) - f(y))) / (FRACT ft) (1 when |ft w| < u), M^-1 into invd
  __device__ static int diag_consume(TS& s, const W& w, int rv, const double (&fr)[N]) {
    bool bad = rv != 0;
    if (!bad) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if (bad) continue;
        const double ft0 = w.at(X_FT + i);
        const double ft = s.h * ft0 - w.zn(1, i);
        double Mi = 1.0;
        if (fabs(ft * w.ewt(i)) >= UROUND) Mi = (FRACT * ft + (-s.h) * (fr[i] - ft0)) / (FRACT * ft);
        if (Mi == 0.0) {
          bad = true;
        } else {
          w.invd(i) = 1.0 / Mi;
        }
      }
      w.at(X_GSV) = s.gamma;
    }
    I::setup_done(s);
    return bad ? I::A_NFAIL : I::A_SOLVE;
  }
  // CVDiagSolve: M^-1 updated exactly when gamma moved since the setup; delta = M^-1 (-G) (no 2/(1+gamrat))
  __device__ static int diag_solve(TS& s, const W& w) {
    s.nni++;
    const double gsv = w.at(X_GSV);
    if (gsv != s.gamma) {
      const double r = s.gamma / gsv;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double Mi = (1.0 / w.invd(i) + (-1.0)) * r + 1.0;
        if (Mi == 0.0) return I::A_NFAIL;
        w.invd(i) = 1.0 / Mi;
      }
      w.at(X_GSV) = s.gamma;
    }
    double b[N];
#pragma unroll
    for (int i = 0; i < N; ++i) b[i] = (-w.del(i)) * w.invd(i);
    return newton_update(s, w, b);
  }

  // ---- inexact Newton-Krylov (LS_GMRES; oracle lsolve_gmres + orc_gmres, reading R29) ----------
  // Scaled GMRES on A = I - gamma J with S1 = S2 = diag(ewt), J v by a difference quotient of the RHS at the
  // Newton iterate ycur = zn0 + ycor: one K_rhs request per Krylov iteration (phase PH_KRY).
  __device__ static double& Hm(const W& w, int i, int j) { return w.at(X_H + i * KMAXL + j); }
  // request f(ycur + sigma v), v = V_l / ewt (a fresh sigma = 1 / ||v||_WRMS when `fresh`)
  __device__ static int kry_request(TS& s, const W& w, int l, bool fresh) {
    double sig = w.at(X_SIG);
    if (fresh) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double v = w.at(X_V + l * N + i) / w.ewt(i);
        const double p = v * w.ewt(i);
        acc = acc + p * p;
      }
      sig = 1.0 / sqrt(acc / (double)N);
      w.at(X_SIG) = sig;
      w.at(X_DQ) = 0.0;
      w.at(X_L) = (double)l;
      w.at(X_NLI) = w.at(X_NLI) + 1.0;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double v = w.at(X_V + l * N + i) / w.ewt(i);
      w.yq(i) = sig * v + (w.zn(0, i) + w.acor(i));
    }
    s.tq_req = s.tn;
    s.phase = PH_KRY;
    return I::A_RET;
  }
  // x = S2^-1 sum_k y_k V_k from the rotated least-squares system (SUNQRsol), then the Newton update
  __device__ static int kry_finish(TS& s, const W& w, int kdim) {
    double g[KMAXL + 1];
    g[0] = w.at(X_BETA);
#pragma unroll
    for (int i = 1; i <= KMAXL; ++i) g[i] = 0.0;
#pragma unroll
    for (int j = 0; j < KMAXL; ++j) {
      if (j < kdim) {
        const double c = w.at(X_GIV + 2 * j), sn = w.at(X_GIV + 2 * j + 1);
        const double t1 = g[j], t2 = g[j + 1];
        g[j] = c * t1 - sn * t2;
        g[j + 1] = sn * t1 + c * t2;
      }
    }
#pragma unroll
    for (int j = KMAXL - 1; j >= 0; --j) {
      if (j < kdim) {
        const double hjj = Hm(w, j, j);
        if (hjj == 0.0) return I::A_NFAIL;         // QRSOL_FAIL: recoverable
        g[j] = g[j] / hjj;
#pragma unroll
        for (int i = 0; i < KMAXL; ++i)
          if (i < j) g[i] = g[i] - g[j] * Hm(w, i, j);
      }
    }
    double b[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double xc = 0.0;
#pragma unroll
      for (int k = 0; k < KMAXL; ++k)
        if (k < kdim) xc = xc + g[k] * w.at(X_V + k * N + i);
      b[i] = xc / w.ewt(i);
    }
    return newton_update(s, w, b);
  }
  // cvLsSolve (iterative): the small-residual exit, else GMRES from x0 = 0 with V0 = S1 b / beta
  __device__ static int kry_start(TS& s, const W& w) {
    s.nni++;
    const double deltar = EPLIFAC * s.tol;
    double b[N];
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      b[i] = -w.del(i);
      const double p = b[i] * w.ewt(i);
      acc = acc + p * p;
    }
    if (sqrt(acc / (double)N) <= deltar) {
      if (s.m > 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) b[i] = 0.0;
      }
      return newton_update(s, w, b);
    }
    const double delta = deltar * sqrt((double)N);
    double bt = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double v = w.ewt(i) * b[i];
      w.at(X_V + i) = v;
      w.at(X_FY + i) = w.fr(i);
      bt = bt + v * v;
    }
    const double beta = sqrt(bt);
    if (beta <= delta) {       // SUCCESS with x = 0
#pragma unroll
      for (int i = 0; i < N; ++i) b[i] = 0.0;
      return newton_update(s, w, b);
    }
#pragma unroll
    for (int i = 0; i < (KMAXL + 1) * KMAXL; ++i) w.at(X_H + i) = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) w.at(X_V + i) = (1.0 / beta) * w.at(X_V + i);
    w.at(X_BETA) = beta;
    w.at(X_ROT) = 1.0;
    return kry_request(s, w, 0, true);
  }
  // one Krylov iteration with the Jv RHS value fr: V_{l+1} = S1 (v - gamma Jv), MGS (SUNModifiedGS),
  // Givens update (SUNQRfact), rotation residual test (Eq. 6); next request, or the solution
  __device__ static int kry_consume(TS& s, const W& w, int rv, const double (&fr)[N], int maxl) {
    const int l = (int)w.at(X_L);
    if (rv) {                                        // cvLsDQJtimes: shrink sigma and retry
      const double dq = w.at(X_DQ) + 1.0;
      if (dq >= (double)MAX_DQITERS) return I::A_NFAIL;
      w.at(X_DQ) = dq;
      w.at(X_SIG) = w.at(X_SIG) * 0.25;
      return kry_request(s, w, l, false);
    }
    const int k = l + 1;
    double t[N];   // the new Krylov vector V_{l+1}, kept in registers through MGS (memory only at the end)
    {
      const double siginv = 1.0 / w.at(X_SIG);
      const double gm = s.gamma;
      double vk = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double jv = (fr[i] - w.at(X_FY + i)) * siginv;
        const double v = w.at(X_V + l * N + i) / w.ewt(i);
        const double z = v - gm * jv;
        t[i] = w.ewt(i) * z;
        vk = vk + t[i] * t[i];
      }
      // modified Gram-Schmidt against V_0..V_l, with the re-orthogonalisation test (FACTOR 1000)
      const double vk_norm = sqrt(vk);
      for (int i0 = 0; i0 < k; ++i0) {
        double vi[N];
#pragma unroll
        for (int j = 0; j < N; ++j) vi[j] = w.at(X_V + i0 * N + j);
        double h = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) h = h + vi[j] * t[j];
        Hm(w, i0, l) = h;
#pragma unroll
        for (int j = 0; j < N; ++j) t[j] = t[j] + (-h) * vi[j];
      }
      double nv2 = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) nv2 = nv2 + t[j] * t[j];
      double nv = sqrt(nv2);
      double temp = 1000.0 * vk_norm;
      if ((temp + nv) == temp) {
        double nn2 = 0.0;
        for (int i0 = 0; i0 < k; ++i0) {
          double vi[N];
#pragma unroll
          for (int j = 0; j < N; ++j) vi[j] = w.at(X_V + i0 * N + j);
          double np = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) np = np + vi[j] * t[j];
          temp = 1000.0 * Hm(w, i0, l);
          if ((temp + np) == temp) continue;
          Hm(w, i0, l) = Hm(w, i0, l) + np;
#pragma unroll
          for (int j = 0; j < N; ++j) t[j] = t[j] + (-np) * vi[j];
          nn2 = nn2 + np * np;
        }
        if (nn2 != 0.0) {
          const double np = nv * nv - nn2;
          nv = (np > 0.0) ? sqrt(np) : 0.0;
        }
      }
      Hm(w, k, l) = nv;
    }
    // Givens: the previous rotations on column l, then a new one zeroing H[l+1][l]
    for (int j = 0; j < l; ++j) {
      const double c = w.at(X_GIV + 2 * j), sn = w.at(X_GIV + 2 * j + 1);
      const double t1 = Hm(w, j, l), t2 = Hm(w, j + 1, l);
      Hm(w, j, l) = c * t1 - sn * t2;
      Hm(w, j + 1, l) = sn * t1 + c * t2;
    }
    const double t1 = Hm(w, l, l), t2 = Hm(w, l + 1, l);
    double c, sn;
    if (t2 == 0.0) {
      c = 1.0;
      sn = 0.0;
    } else if (fabs(t2) >= fabs(t1)) {
      const double t3 = t1 / t2;
      sn = -1.0 / sqrt(1.0 + t3 * t3);
      c = -sn * t3;
    } else {
      const double t3 = t2 / t1;
      c = 1.0 / sqrt(1.0 + t3 * t3);
      sn = -c * t3;
    }
    w.at(X_GIV + 2 * l) = c;
    w.at(X_GIV + 2 * l + 1) = sn;
    const double hll = c * t1 - sn * t2;
    Hm(w, l, l) = hll;
    if (hll == 0.0) return I::A_NFAIL;                 // QRFACT_FAIL: recoverable
    const double rot = w.at(X_ROT) * sn;
    w.at(X_ROT) = rot;
    const double beta = w.at(X_BETA);
    const double rho = fabs(rot * beta);
    const double delta = EPLIFAC * s.tol * sqrt((double)N);
    if (rho <= delta) return kry_finish(s, w, k);
    if (k >= maxl) {   // cap: RES_REDUCED accepted on the first Newton iteration only (cvLsSolve)
      if (rho < beta && s.m == 0) return kry_finish(s, w, k);
      return I::A_NFAIL;
    }
    const double inv = 1.0 / Hm(w, k, l);
#pragma unroll
    for (int j = 0; j < N; ++j) w.at(X_V + k * N + j) = inv * t[j];
    return kry_request(s, w, k, true);
  }

  // the trip after the setup decision (both passes): SOLVE .. ATTEMPT, in the
  // stage order of TpcIntegrator::trip.  Returns A_RET (RHS requested) or A_DONE.
  // DEFER_STORE: a finished cell is not stored here; it is marked PH_STORE and returns A_STORE (K_init
  // stores it and loads the next cell with full warps)
  template <bool DEFER_STORE = false>
  __device__ static int finish(const Opts& o, TS& s, const W& w, int act, const double* lu, double* y,
                               const double* fext, const double* aux, const double* atol,
                               unsigned long long* counter, Agg& acc, const CellStatsPtrs& cs) {
    if (act == I::A_SOLVE) {
      if constexpr (LS == LS_DENSE) act = solve(s, w, lu);
      else if constexpr (LS == LS_DIAG) act = diag_solve(s, w);
      else act = kry_start(s, w);
    }
    if (act == I::A_NFAIL) act = I::nfail(o, s, w);
    if (act == I::A_ERRTEST) act = I::errtest(o, s, w);
    if (act == I::A_STEP_TOP) act = I::step_top(o, s, w);
    if (DEFER_STORE && act == I::A_STORE) {
      s.phase = PH_STORE;
      return act;
    }
    if (act == I::A_STORE) {
      if constexpr (LS == LS_GMRES) {   // the cell's linear iterations (aggregate only), reset for the next cell
        if (s.status != ST_NONFINITE) atomicAdd(&acc.nli, (unsigned long long)w.at(X_NLI));
        w.at(X_NLI) = 0.0;
      }
      I::store(o, s, w, y, acc, cs);
      act = I::A_LOAD;
    }
    if (act == I::A_LOAD) act = I::load(o, s, w, y, fext, aux, atol, counter, acc, cs);
    if (act == I::A_ATTEMPT) act = I::attempt(o, s, w, atol);
    return act;
  }
};

// initialise the pool: every slot empty (phase DONE)
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void split_init_kernel(SplitBufs b) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s == 0) {
    b.live[0] = b.live[1] = 0;
    for (int i = 0; i < 6; ++i) b.cnt[i] = 0;
  }
  if (s >= b.slots) return;
  TS* t = Split<Mech, GM, LS>::ts(b, s);
  if constexpr (LS == LS_GMRES) Split<Mech, GM, LS>::ws(b, s).at(Split<Mech, GM, LS>::X_NLI) = 0.0;
  t->phase = PH_DONE;
  t->flag = 0;
  t->pend = 0;
  b.rv[s] = 0;
}

// ------------------------------------------------------------------ K_ctl
// one trip of every slot (slot = block * BLOCK + thread); the block's TS
// records are copied through shared memory (coalesced).  A cell whose last
// trip stopped at a matrix setup (phase PH_SETUP) resumes after it: the setup
// kernels ran in between, so the trip costs the cell one extra iteration
// (its RHS slot idles once) instead of a latency-bound second pass.
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_CTL_BLOCK, (Mech::N > 32 ? 2 : BDFB_SPLIT_CTL_MINB))   // n = 54: 255 registers measured 12% faster
    split_ctl_kernel(Opts o, SplitBufs b, int it, double* y, const double* fext, const double* aux,
                     const double* atol, unsigned long long* counter, Agg* agg, CellStatsPtrs cs) {
  using SP = Split<Mech, GM, LS>;
  using I = typename SP::I;
  constexpr int N = Mech::N;
  extern __shared__ double smem[];           // TS records of the block's threads (TS_STRIDE each)
  // every shared structure of K_ctl is warp-private (TS staging, statistics): no block barrier, so a warp whose
  // lanes finish early leaves without waiting for the block's slowest warp (ncu: block barriers were ~10% of
  // the stall cycles); atol is read through L1 from global memory
  __shared__ Agg wacc[BDFB_SPLIT_CTL_BLOCK / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) wacc[warp] = Agg{};
  unsigned* cnt = b.cnt + 3 * (it & 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // the next iteration's lists and live count (their last
    unsigned* nx = b.cnt + 3 * ((it + 1) & 1);   // readers, iteration it - 1, have finished)
    nx[0] = nx[1] = nx[2] = 0;
    b.live[(it + 1) & 1] = 0;
  }
  // the warp's 32 TS records are contiguous in HBM: stage them through shared memory (coalesced), warp-local
  const long long w0 = (long long)blockIdx.x * BDFB_SPLIT_CTL_BLOCK + (threadIdx.x & ~31u);
  const long long nrec = (b.slots - w0 < 32 ? (b.slots - w0 > 0 ? b.slots - w0 : 0) : 32) * TS_STRIDE;
#if BDFB_SPLIT_TS_SMEM
  double* wsm = smem + (threadIdx.x & ~31u) * TS_STRIDE;
  {
    const double* src = b.ts + w0 * TS_STRIDE;
    if (nrec == 32 * TS_STRIDE) {   // full warp: all 16-byte loads in flight at once (one HBM round trip)
      constexpr int NV2 = 32 * TS_STRIDE / 2;   // TS_STRIDE odd: 32 records = an even number of doubles
      const double2* s2 = reinterpret_cast<const double2*>(src);
      double2* d2 = reinterpret_cast<double2*>(wsm);
      double2 v[(NV2 + 31) / 32];
#pragma unroll
      for (int k = 0; k < (NV2 + 31) / 32; ++k)
        if (lane + 32 * k < NV2) v[k] = s2[lane + 32 * k];
#pragma unroll
      for (int k = 0; k < (NV2 + 31) / 32; ++k)
        if (lane + 32 * k < NV2) d2[lane + 32 * k] = v[k];
    } else {
      for (long long i = lane; i < nrec; i += 32) wsm[i] = src[i];
    }
  }
#endif
  const long long slot = w0 + lane;
  const bool have = slot < b.slots;
#if BDFB_SPLIT_PREFETCH
  // bulk L2 prefetch (one TMA instruction each) of the warp's 32 LU records and of its state rows: the
  // Newton solve's column loads and the Nordsieck passes then hit L2 instead of waiting on HBM
  // (3: the warp's Nordsieck rows only, 4: its Nordsieck, weight, correction and request rows -- the rows the
  // ATTEMPT pass and the residual read, 6 n resp. 9 n elements x 256 B)
  if (lane == 0 && w0 + 32 <= b.slots) {
#if BDFB_SPLIT_PREFETCH <= 2
    const double* lu0 = SP::lurec(b, w0);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lu0), "r"((unsigned)(32 * SP::LUREC * 8)) : "memory");
#endif
#if BDFB_SPLIT_PREFETCH == 2
    const double* v0 = b.vec + ((w0 >> 5) * SP::D) * 32;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v0), "r"((unsigned)(SP::D * 32 * 8)) : "memory");
#elif BDFB_SPLIT_PREFETCH >= 3
    constexpr int ROWS = BDFB_SPLIT_PREFETCH == 3 ? (QMAX + 1) * N : SP::W::O_DEL;
    const double* v0 = b.vec + ((w0 >> 5) * SP::D) * 32;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(v0), "r"((unsigned)(ROWS * 32 * 8)) : "memory");
#endif
  }
#endif
  __syncwarp();   // the warp's staged TS records, wacc
#if BDFB_SPLIT_TS_SMEM
  TS& s = *reinterpret_cast<TS*>(smem + threadIdx.x * TS_STRIDE);
#else
  TS& s = *SP::ts(b, have ? slot : 0);
#endif
  const typename SP::W w = SP::ws(b, have ? slot : 0);
  const double* lu = SP::lurec(b, have ? slot : 0);
  int act = I::A_DONE;
  bool setup = false, jreq = false, init = false;
  if (have) {
    bool run = true;
    if (s.phase == PH_DONE) {   // empty slot: live only while the work counter has cells left
      const unsigned long long next = *reinterpret_cast<volatile unsigned long long*>(counter);
      run = next < (unsigned long long)o.ncells;
    }
#if BDFB_SPLIT_INIT_KERNEL
    if (run && (s.phase == PH_DONE || s.phase == PH_INIT || s.phase == PH_HIN)) {   // K_init's work
      init = true;
      run = false;
    }
#endif
    if (run && s.phase == PH_SETUP) {   // resume after the setup kernels (TpcIntegrator::trip order)
      act = s.pend;
      if (act == I::A_SETUP_J) {
        if (s.coop) {
          I::setup_done(s);
          act = I::A_NFAIL;
        } else {
          act = I::A_SETUP_LU;
        }
      }
      if (act == I::A_SETUP_LU) {
        I::setup_done(s);
        act = s.coop ? I::A_NFAIL : I::A_SOLVE;
      }
      s.pend = 0;
    } else if (run) {
      double fr[N];
      int rv = 0;
      const int ph = s.phase;
      if (ph == PH_INIT || ph == PH_HIN || ph == PH_NRES || ph == PH_ETF3 || (LS == LS_DIAG && ph == PH_DIAG) ||
          (LS == LS_GMRES && ph == PH_KRY)) {
        rv = b.rv[slot];
        if (ph != PH_KRY) s.nfe++;   // the Jv quotients' RHS calls are not counted in nfe (CVODE's nfeDQ)
        if (LS != LS_DENSE || rv != RV_SOLVED) {
#pragma unroll
          for (int i = 0; i < N; ++i) fr[i] = w.fr(i);
        }
      }
      if (LS == LS_DENSE && rv == RV_SOLVED) {   // consume + SOLVE ran in K_rhs
        act = SP::solved(s, w);
      } else if (LS == LS_DIAG && ph == PH_DIAG) {
        act = SP::diag_consume(s, w, rv, fr);
      } else if (LS == LS_GMRES && ph == PH_KRY) {
        act = SP::kry_consume(s, w, rv, fr, b.maxl);
      } else {
        if (LS == LS_GMRES && ph == PH_NRES && s.m == 0) {   // no setup for matrix-free GMRES: R = 1 per solve,
          s.crate = 1.0;                                     // no matrix refresh, no retry (reading R29)
          s.setup = 0;
          s.jcur = 1;
        }
        act = I::consume(o, s, w, rv, fr);
      }
      if (act == I::A_HIN_FINISH) act = I::hin_finish(o, s);
      if (act == I::A_START) act = I::start(o, s, w);
      if (act == I::A_SETUP) act = (LS == LS_DIAG) ? SP::diag_request(s, w) : I::setup_decide(s);
      if (LS == LS_DENSE && (act == I::A_SETUP_J || act == I::A_SETUP_LU)) {
        s.pend = act;
        s.coop = 0;
        s.phase = PH_SETUP;
        setup = true;
        jreq = act == I::A_SETUP_J;
        act = I::A_RET;      // live; finish() passes A_RET through
      }
    }
    // one call site: lanes that resumed and lanes that consumed an RHS value run the rest together
    if (run) act = SP::template finish<BDFB_SPLIT_INIT_KERNEL != 0>(o, s, w, act, lu, y, fext, aux, atol, counter,
                                                                      wacc[warp], cs);
    if (act == I::A_STORE) init = true;   // deferred store (K_init)
  }
  // setup / Jacobian lists: one atomic per warp and list
  {
    const unsigned bs = __ballot_sync(0xffffffffu, setup), bj = __ballot_sync(0xffffffffu, jreq);
    unsigned os = 0, oj = 0;
    if (lane == 0) {
      if (bs) os = atomicAdd(&cnt[0], __popc(bs));
      if (bj) oj = atomicAdd(&cnt[1], __popc(bj));
    }
    os = __shfl_sync(0xffffffffu, os, 0);
    oj = __shfl_sync(0xffffffffu, oj, 0);
    const unsigned below = (1u << lane) - 1u;
    if (setup) b.slist[os + __popc(bs & below)] = (int)slot;
    if (jreq) b.jlist[oj + __popc(bj & below)] = (int)slot;
    const unsigned bi = __ballot_sync(0xffffffffu, init);
    unsigned oi = 0;
    if (lane == 0 && bi) oi = atomicAdd(&cnt[2], __popc(bi));
    oi = __shfl_sync(0xffffffffu, oi, 0);
    if (init) b.ilist[oi + __popc(bi & below)] = (int)slot;
    const unsigned bl = __ballot_sync(0xffffffffu, act == I::A_RET);
    if (lane == 0 && bl) atomicAdd(&b.live[it & 1], (unsigned long long)__popc(bl));
  }
#if BDFB_SPLIT_TS_SMEM
  __syncwarp();
  {
    double* dst = b.ts + w0 * TS_STRIDE;
#pragma unroll 4
    for (long long i = lane; i < nrec; i += 32) dst[i] = wsm[i];
  }
#endif
  __syncwarp();
  if (lane == 0 && wacc[warp].cells_done) {
    const Agg& a = wacc[warp];
    atomicAdd(&agg->n_failed, a.n_failed);
    atomicAdd(&agg->nst, a.nst);
    atomicAdd(&agg->nfe, a.nfe);
    atomicAdd(&agg->nje, a.nje);
    atomicAdd(&agg->nsetups, a.nsetups);
    atomicAdd(&agg->nni, a.nni);
    atomicAdd(&agg->netf, a.netf);
    atomicAdd(&agg->ncfn, a.ncfn);
    atomicMax(&agg->nst_max, a.nst_max);
    atomicMax(&agg->nfe_max, a.nfe_max);
    atomicAdd(&agg->cells_done, a.cells_done);
    if (LS == LS_GMRES) atomicAdd(&agg->nli, a.nli);
  }
}

// ------------------------------------------------------------------ K_init
// thread per init-list entry (compacted: full warps of cells that start or end): store a finished cell and
// load the next one from the work counter (f(t0, y0) requested), or consume a cvHin RHS value (h0 by cvHin;
// once h0 is set, start, step_top and the first ATTEMPT: the first Newton residual requested).  The state
// is accessed in place (TS record L1-cached; the SoA rows of scattered slots: rare work).
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK) split_init_cells_kernel(Opts o, SplitBufs b, int it, double* y,
                                                                           const double* fext, const double* aux,
                                                                           const double* atol,
                                                                           unsigned long long* counter, Agg* agg,
                                                                           CellStatsPtrs cs) {
  using SP = Split<Mech, GM, LS>;
  using I = typename SP::I;
  constexpr int N = Mech::N;
  __shared__ double satol[N];
  __shared__ Agg wacc[BDFB_SPLIT_BLOCK / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < N) satol[threadIdx.x] = atol[threadIdx.x];
  if (lane == 0) wacc[warp] = Agg{};
  __syncthreads();
  const long long cnt = b.cnt[3 * (it & 1) + 2];
  unsigned long long nlive = 0;
  for (long long e = (long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x; e - lane < cnt;
       e += (long long)gridDim.x * BDFB_SPLIT_BLOCK) {
    int act = I::A_DONE;
    if (e < cnt) {
      const long long slot = b.ilist[e];
      TS& s = *SP::ts(b, slot);
      const typename SP::W w = SP::ws(b, slot);
      const int ph = s.phase;
      if (ph == PH_STORE) {
        I::store(o, s, w, y, wacc[warp], cs);
        act = I::A_LOAD;
      } else if (ph == PH_DONE) {
        act = I::A_LOAD;
      } else {                                   // PH_INIT / PH_HIN: a cvHin RHS value is ready
        double fr[N];
        const int rv = b.rv[slot];
        s.nfe++;
#pragma unroll
        for (int i = 0; i < N; ++i) fr[i] = w.fr(i);
        act = I::consume(o, s, w, rv, fr);
        if (act == I::A_HIN_FINISH) act = I::hin_finish(o, s);
        if (act == I::A_START) act = I::start(o, s, w);
        if (act == I::A_STEP_TOP) act = I::step_top(o, s, w);
        if (act == I::A_STORE) {
          I::store(o, s, w, y, wacc[warp], cs);
          act = I::A_LOAD;
        }
      }
      if (act == I::A_LOAD) act = I::load(o, s, w, y, fext, aux, satol, counter, wacc[warp], cs);
      if (act == I::A_ATTEMPT) act = I::attempt(o, s, w, satol);
    }
    const unsigned bl = __ballot_sync(0xffffffffu, act == I::A_RET);
    if (lane == 0) nlive += __popc(bl);
  }
  if (lane == 0 && nlive) atomicAdd(&b.live[it & 1], nlive);
  if (lane == 0 && wacc[warp].cells_done) {
    const Agg& a = wacc[warp];
    atomicAdd(&agg->n_failed, a.n_failed);
    atomicAdd(&agg->nst, a.nst);
    atomicAdd(&agg->nfe, a.nfe);
    atomicAdd(&agg->nje, a.nje);
    atomicAdd(&agg->nsetups, a.nsetups);
    atomicAdd(&agg->nni, a.nni);
    atomicAdd(&agg->netf, a.netf);
    atomicAdd(&agg->ncfn, a.ncfn);
    atomicMax(&agg->nst_max, a.nst_max);
    atomicMax(&agg->nfe_max, a.nfe_max);
    atomicAdd(&agg->cells_done, a.cells_done);
  }
}

// ------------------------------------------------------------------ K_jac
// one cell per group of G lanes (lane i = component i): the analytic Jacobian
// of the group model (mech_model.cuh: lanes over species and reactions), row
// i into the cell's column-major J record; status -> TS.coop (nonzero:
// recoverable failure).  Shared scratch per group: RHS scratch SG + the
// Jacobian's per-reaction partials JG.
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK) split_jac_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  constexpr int N = Mech::N, G = GM::G;
  constexpr int MS = N | 1;                      // odd row stride of the shared J (conflict-free)
  extern __shared__ double smem[];
  Grp<G> g;
  const int gi = threadIdx.x / G;
  double* sc = smem + gi * (GM::SG + GM::JG + N * MS);
  double* jm = sc + GM::SG + GM::JG;
  const long long cnt = b.cnt[3 * (it & 1) + 1], groups = (long long)gridDim.x * (BDFB_SPLIT_BLOCK / G);
  for (long long e = ((long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x) / G; e < cnt; e += groups) {
    const long long slot = b.jlist[e];
    const typename SP::W w = SP::ws(b, slot);
    TS* t = SP::ts(b, slot);
    const double yv = g.lane < N ? w.yq(g.lane) : 0.0;
    double* J = b.J + slot * SP::JREC;
    const int r = GM::template jac<MS>(g, yv, t->aux, jm + (g.lane < N ? g.lane : 0), sc, sc + GM::SG);
    g.sync();
    if (!r && g.lane < N) {
#pragma unroll 2
      for (int j = 0; j < N; ++j) J[j * N + g.lane] = jm[j * MS + g.lane];
    }
    if (g.lane == 0) t->coop = r;
    g.sync();
  }
}

// K_jac variant: one thread per Jacobian-list entry, the generated straight-line column-major Jacobian
// (gen/tpc_<mech>.cuh jac_cm) reading yq from VEC (stride 32) into the slot's J record, scratch in its LU record
// (K_lu overwrites it right after).  Selected with BDFB_SPLIT_JAC_TPC=1 (measurement).
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK) split_jac_tpc_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  const long long cnt = b.cnt[3 * (it & 1) + 1];
  for (long long e = (long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x; e < cnt;
       e += (long long)gridDim.x * BDFB_SPLIT_BLOCK) {
    const long long slot = b.jlist[e];
    const typename SP::W w = SP::ws(b, slot);
    TS* t = SP::ts(b, slot);
    t->coop = Mech::template jac_cm<VEC_S>(&w.yq(0), t->aux, b.J + slot * SP::JREC, SP::lurec(b, slot));
  }
}

// K_jac in two passes (default for n <= 32 when the scratch fits the LU record): the generated jac_cm split
// into pass 1, one thread per Jacobian-list entry (thermo, every reaction's kf, kr, dq/dT, dq/d[M], the energy
// sums; gen/tpc_<mech>.cuh jac_p1) into a warp-blocked SoA scratch indexed by the list position (pass 1 stores
// and pass 2 loads are one 256-byte line per warp), and pass 2, one thread per (entry, column j) with j
// warp-uniform and column-major across warps (each warp of a block runs the same column's code), writing
// column j of the J record (jac_col).  Same operations as jac_cm.  The
// Jacobian list of one iteration is ~10^4 cells: one thread per cell leaves most of the GPU idle behind one
// serial chain (the group/lanes K_jac: ~53K warp instructions per Jacobian, ncu profiles/r2).
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK) split_jac_p1_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  const long long cnt = b.cnt[3 * (it & 1) + 1];
  for (long long e = (long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x; e < cnt;
       e += (long long)gridDim.x * BDFB_SPLIT_BLOCK) {
    const long long slot = b.jlist[e];
    const typename SP::W w = SP::ws(b, slot);
    TS* t = SP::ts(b, slot);
    t->coop = Mech::template jac_p1<VEC_S, 32>(&w.yq(0), t->aux, b.jscr + ((e >> 5) * Mech::NSC2) * 32 + (e & 31));
    static_assert(Mech::NSC2 <= Mech::NSC3, "scratch");
  }
}
// K_jac pass 1 parted (default): thread per (entry, part P) with P warp-uniform and equal for neighbour warps
// (jac_part: the reactions dealt round-robin to Mech::NPART parts), then jac_sum, one thread per entry (the
// per-species thermo, the production rates added in part order, the energy sums and scalars): NPART x the
// threads of split_jac_p1_kernel over NPART x shorter chains (ncu: p1 ran ~2 warps per SM, IPC 0.3)
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK) split_jac_part_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  const long long cnt = b.cnt[3 * (it & 1) + 1];
  const long long neb = (cnt + 31) / 32;
  const int lane = threadIdx.x & 31;
  const long long nw = neb * Mech::NPART, wstride = ((long long)gridDim.x * BDFB_SPLIT_BLOCK) >> 5;
  for (long long gw = ((long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x) >> 5; gw < nw; gw += wstride) {
    const int P = (int)(gw / neb);
    const long long e = (gw - P * neb) * 32 + lane;
    if (e >= cnt) continue;
    const long long slot = b.jlist[e];
    const typename SP::W w = SP::ws(b, slot);
    TS* t = SP::ts(b, slot);
    const int rv = Mech::template jac_part<VEC_S, 32>(P, &w.yq(0), t->aux,
                                                       b.jscr + ((e >> 5) * Mech::NSC3) * 32 + (e & 31));
    if (P == 0) t->coop = rv;
  }
}
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK) split_jac_sum_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  const long long cnt = b.cnt[3 * (it & 1) + 1];
  for (long long e = (long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x; e < cnt;
       e += (long long)gridDim.x * BDFB_SPLIT_BLOCK) {
    const long long slot = b.jlist[e];
    const TS* t = SP::ts(b, slot);
    if (t->coop) continue;
    const typename SP::W w = SP::ws(b, slot);
    Mech::template jac_sum<VEC_S, 32>(&w.yq(0), t->aux, b.jscr + ((e >> 5) * Mech::NSC3) * 32 + (e & 31));
  }
}
#ifndef BDFB_SPLIT_JAC_PARTS
#define BDFB_SPLIT_JAC_PARTS 1   // 0: pass 1 one thread per entry (split_jac_p1_kernel)
#endif
// scratch stride (doubles per entry) of the two-pass Jacobian
template <class Mech>
__host__ __device__ constexpr int jac_scr_doubles() { return BDFB_SPLIT_JAC_PARTS ? Mech::NSC3 : Mech::NSC2; }

template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK) split_jac_p2_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  constexpr int N = Mech::N;
  const long long cnt = b.cnt[3 * (it & 1) + 1];
  const long long neb = (cnt + 31) / 32;                       // 32-entry blocks
  const int lane = threadIdx.x & 31;
  const long long nw = neb * N, wstride = ((long long)gridDim.x * BDFB_SPLIT_BLOCK) >> 5;
  for (long long gw = ((long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x) >> 5; gw < nw; gw += wstride) {
    const int j = (int)(gw / neb);                             // column: warp-uniform, equal for neighbour warps
    const long long e = (gw - j * neb) * 32 + lane;
    if (e >= cnt) continue;
    const long long slot = b.jlist[e];
    if (SP::ts(b, slot)->coop) continue;                       // pass 1 failed (T <= 0): recoverable
    Mech::template jac_col<32>(j, b.jscr + ((e >> 5) * jac_scr_doubles<Mech>()) * 32 + (e & 31),
                               b.J + slot * SP::JREC);
  }
}

// ------------------------------------------------------------------ K_dqjac
// Difference-quotient Jacobian (CVODE's cvLsDenseDQJac, the paper's approaches 3A/3B; SURVEY row
// f1), one thread per (Jacobian-list entry, column j): the cell's J is evaluated at yq = zn[0] with
// fy = the consumed RHS value (fr row); srur = sqrt(u), fnorm = ||fy||_WRMS (sequential, R15 G = 1),
// minInc = 1000 |h| u n fnorm (1 if fnorm = 0), inc = max(srur |y_j|, minInc / ewt_j),
// J(:, j) = (1/inc) f(y + inc e_j) + (-(1/inc)) fy, f = the generated RHS + F -- the oracle's orc_jac_dq
// operation for operation.  An RHS failure marks the cell (TS.coop = 1: a recoverable setup failure).
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK, 3) split_dqjac_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  constexpr int N = Mech::N;
  const long long cnt = (long long)b.cnt[3 * (it & 1) + 1] * N, stride = (long long)gridDim.x * BDFB_SPLIT_BLOCK;
  for (long long t = (long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x; t < cnt; t += stride) {
    const long long e = t / N;
    const int j = (int)(t - e * N);
    const long long slot = b.jlist[e];
    const typename SP::W w = SP::ws(b, slot);
    TS* ts = SP::ts(b, slot);
    double y[N], fy[N], ft[N];
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      y[i] = w.yq(i);
      fy[i] = w.fr(i);
      const double p = fy[i] * w.ewt(i);
      acc = acc + p * p;
    }
    const double fnorm = sqrt(acc / (double)N);
    const double minInc = (fnorm != 0.0) ? (1000.0 * fabs(ts->h) * UROUND * N * fnorm) : 1.0;
    double yj = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (i == j) yj = y[i];
    const double inc = fmax(sqrt(UROUND) * fabs(yj), minInc / w.ewt(j));
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (i == j) y[i] = yj + inc;
    const int rv = Mech::rhs(y, ts->aux, ft);
    if (rv) {
      ts->coop = 1;
      continue;
    }
    const double inc_inv = 1.0 / inc;
    double* Jc = b.J + slot * SP::JREC + (long long)j * N;
#pragma unroll
    for (int i = 0; i < N; ++i) Jc[i] = inc_inv * (ft[i] + w.fext(i)) + (-inc_inv) * fy[i];
  }
}

// ------------------------------------------------------------------ K_lu
// One cell per group of 8 lanes, 4 cells per warp.  Lane l of the group holds
// rows r = l + 8 s (s < R = ceil(n/8)) of M = I - gamma J in registers; rows
// never move between lanes, each tracks its LAPACK position pos (as
// coop_factor).  Per column k: the first index (in position order) of the
// max |.| over positions >= k by a 3-step xor butterfly, the pivot row's
// entries broadcast by shuffles, 1/pivot once, multipliers m = a_ik (1/pv)
// and fma updates -- the listing's LU_FACTOR operation for operation
// (reading R16), so pivots and factors are bit-identical to the oracle.
// Versus one cell per warp (coop_factor) every shuffle of the pivot row
// serves 4 cells and every lane has ~3 rows of FMAs: ~4x fewer instructions
// per factorisation.
// The whole warp runs every column together (full-mask shuffles, no early exit): a shuffle with a per-group
// mask compiled to a convergence barrier around every SHFL (WARPSYNC + BSSY/BSYNC + ENDCOLLECTIVE: 3.1K of the
// kernel's 19K SASS instructions, ncu IPC 1.4, 2.4K warp instructions per LU).  A group whose pivot is an exact
// zero keeps computing on garbage that is never stored; info = k + 1 of its first zero pivot, else 0.
constexpr int OCT = 8;
// a[ps][j] for a runtime slot ps < R (a chain of R - 1 selects: the pivot row is always a real row, so the last
// slot needs no test; the zero-initialised form cost R selects per double -- 41% of K_lu's instructions were FSEL)
template <int R, int NN>
__device__ __forceinline__ double oct_pick(const double (&a)[R][NN], int ps, int j) {
  double v = a[R - 1][j];
#pragma unroll
  for (int s = R - 2; s >= 0; --s) v = (ps == s) ? a[s][j] : v;
  return v;
}

// column k of oct_factor (k a compile-time constant so that a[][] stays in registers)
template <int N, int K>
__device__ __forceinline__ void oct_column(int gl, double (&a)[(N + OCT - 1) / OCT][N], int (&pos)[(N + OCT - 1) / OCT],
                                           double (&dinv)[(N + OCT - 1) / OCT], int& info) {
  constexpr int R = (N + OCT - 1) / OCT;
  // local candidate: max |a[s][K]| over owned rows with pos >= K, ties -> smaller pos; (pos, row) packed in one
  // int (pos in the high half: positions are distinct, so packed order = position order)
  double bv = -1.0;
  int bpr = 0x7fffffff;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int r = gl + OCT * s;
    if (r < N && pos[s] >= K) {
      const double v = fabs(a[s][K]);
      const int pr = (pos[s] << 16) | r;
      if (v > bv || (v == bv && pr < bpr)) {
        bv = v;
        bpr = pr;
      }
    }
  }
#pragma unroll
  for (int off = OCT / 2; off >= 1; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, off, OCT);
    const int opr = __shfl_xor_sync(0xffffffffu, bpr, off, OCT);
    if (ov > bv || (ov == bv && opr < bpr)) {
      bv = ov;
      bpr = opr;
    }
  }
  if (!(bv > 0.0) && info == 0) info = K + 1;   // exact zero pivot (uniform in the group)
  const int bp = bpr >> 16, br = bpr & 0xffff;
  const int pl = br & (OCT - 1), ps = br / OCT;   // owner lane and slot of the pivot row
  const double pv = __shfl_sync(0xffffffffu, oct_pick<R>(a, ps, K), pl, OCT);
  const double rinv = 1.0 / pv;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int r = gl + OCT * s;
    if (r == br) {
      pos[s] = K;
      dinv[s] = rinv;
    } else if (pos[s] == K) {
      pos[s] = bp;
    }
  }
  // multipliers; rows that take no update this column (already pivoted, or padding) get m = 0, so the update
  // below is one unpredicated DFMA per row: fma(-0, pj, a) = a (for finite pj; a -0.0 entry may become +0.0,
  // equal as a number -- reading R16 note in DESIGN.md) instead of a DFMA and two selects
  double m[R];
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const bool upd = (gl + OCT * s < N) && pos[s] > K;
    const double mk = a[s][K] * rinv;
    m[s] = upd ? mk : 0.0;
    if (upd) a[s][K] = mk;
  }
#pragma unroll
  for (int j = K + 1; j < N; ++j) {
    const double pj = __shfl_sync(0xffffffffu, oct_pick<R>(a, ps, j), pl, OCT);
#pragma unroll
    for (int s = 0; s < R; ++s)
      if (gl + OCT * s < N) a[s][j] = fma(-m[s], pj, a[s][j]);
  }
}

template <int N, int... Ks>
__device__ __forceinline__ void oct_columns(int gl, double (&a)[(N + OCT - 1) / OCT][N], int (&pos)[(N + OCT - 1) / OCT],
                                            double (&dinv)[(N + OCT - 1) / OCT], int& info,
                                            std::integer_sequence<int, Ks...>) {
  (oct_column<N, Ks>(gl, a, pos, dinv, info), ...);   // left to right
}

// called by all 32 lanes of the warp together (4 groups); returns 0 or k + 1 of the group's first zero pivot
template <int N>
__device__ __forceinline__ int oct_factor(int gl, double (&a)[(N + OCT - 1) / OCT][N], int (&pos)[(N + OCT - 1) / OCT],
                                          double (&dinv)[(N + OCT - 1) / OCT]) {
  constexpr int R = (N + OCT - 1) / OCT;
  static_assert(N < (1 << 15), "packed (pos, row)");
#pragma unroll
  for (int s = 0; s < R; ++s) {
    pos[s] = gl + OCT * s;
    dinv[s] = 0.0;
  }
  int info = 0;
  oct_columns<N>(gl, a, pos, dinv, info, std::make_integer_sequence<int, N>{});
  return info;
}

// K_lu: one setup-list entry per group of 8 lanes (grid-stride, warp-uniform trips: a group without an entry,
// or whose Jacobian failed, factors the identity and stores nothing); M = I - gamma J from the cell's
// column-major J, oct_factor, factors stored column-major in pivoted row order + 1/U_kk + perm, as the Newton
// solve reads them.
template <class Mech, class GM, int LS = LS_DENSE>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK, 3) split_lu_kernel(SplitBufs b, int it) {   // 12 warps/SM
  using SP = Split<Mech, GM, LS>;
  constexpr int N = Mech::N, R = (N + OCT - 1) / OCT;
  const int lane = threadIdx.x & 31, gl = lane & (OCT - 1);
  const long long cnt = b.cnt[3 * (it & 1)], groups = (long long)gridDim.x * (BDFB_SPLIT_BLOCK / OCT);
  // CTA-uniform trip condition and branch-free entry loads, so that the compiler can prove the warp converged
  // at every shuffle (no BRA.DIV guard splitting the column code into basic blocks)
  for (long long e0 = (long long)blockIdx.x * (BDFB_SPLIT_BLOCK / OCT); e0 < cnt; e0 += groups) {
    const long long e = e0 + threadIdx.x / OCT;
    const bool have = e < cnt;
    const long long slot = b.slist[have ? e : cnt - 1];
    TS* t = SP::ts(b, slot);
    const bool work = have && t->coop == 0;    // the Jacobian failed: the resumed trip handles it
    const double gm = t->gamma;
    const double* J = b.J + slot * SP::JREC;
    double* lu = SP::lurec(b, slot);
    double a[R][N];
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int r = gl + OCT * s;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double v = (r == j ? 1.0 : 0.0) - gm * J[j * N + (r < N ? r : 0)];
        a[s][j] = (r < N) ? (work ? v : (r == j ? 1.0 : 0.0)) : 0.0;
      }
    }
    int pos[R];
    double dinv[R];
    const int info = oct_factor<N>(gl, a, pos, dinv);
    if (work && !info) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int r = gl + OCT * s;
        if (r < N) {
#pragma unroll
          for (int j = 0; j < N; ++j) lu[(j * N + pos[s]) * LU_STRIDE] = a[s][j];
          lu[(SP::LU_INVD + pos[s]) * LU_STRIDE] = dinv[s];
          if (LU_STRIDE == 1) reinterpret_cast<int*>(lu + SP::LU_PERM)[pos[s]] = r;
          else lu[(SP::LU_PERM + pos[s]) * LU_STRIDE] = (double)r;
        }
      }
    }
    __syncwarp();
    if (work && gl == 0) t->coop = info;
  }
}

// ------------------------------------------------------------------ K_rhs
// thread per slot: fr = R(yq) + F for a pending RHS request.
#ifndef BDFB_SPLIT_RHS_MINB
#define BDFB_SPLIT_RHS_MINB 3   // 168 registers, 12 warps/SM: 7% faster than 255 registers / 8 warps (measured)
#endif
// VAR 0: 128-thread blocks, 3 per SM, free-running warps; VAR 1: the same with a block barrier per
// grid-stride trip; VAR 2: one 384-thread block per SM with a barrier per trip, so that all 12 warps of an SM
// walk the ~10K-instruction generated RHS together (instruction-cache locality; see erk.cu)
// VAR 3: VAR 0 with e^{-g/RT} and its reciprocals in shared memory (rhs_sm: 2K fewer live registers)
template <int VAR>
struct RhsVar {
  static constexpr int BLOCK = VAR == 2 ? 384 : BDFB_SPLIT_BLOCK;
  static constexpr int MINB = VAR == 2 ? 1 : (VAR == 4 ? 4 : BDFB_SPLIT_RHS_MINB);   // VAR 4: VAR 3 at 16 warps/SM
  static constexpr bool SYNC = VAR == 1 || VAR == 2;
  static constexpr bool SM = VAR == 3 || VAR == 4;
};
template <class Mech, class GM, int LS = LS_DENSE, int VAR = 0>
__global__ void __launch_bounds__(RhsVar<VAR>::BLOCK, RhsVar<VAR>::MINB) split_rhs_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  using V = RhsVar<VAR>;
  constexpr int N = Mech::N;
  const long long stride = (long long)gridDim.x * V::BLOCK;
  for (long long s0 = (long long)blockIdx.x * V::BLOCK; s0 < b.slots; s0 += stride) {   // block-uniform trips
    if (V::SYNC) __syncthreads();
    const long long slot = s0 + threadIdx.x;
    if (slot >= b.slots) continue;
    const TS* t = SP::ts(b, slot);
    const int ph = t->phase;
    if (!(ph == PH_INIT || ph == PH_HIN || ph == PH_NRES || ph == PH_ETF3 || (LS == LS_DIAG && ph == PH_DIAG) ||
          (LS == LS_GMRES && ph == PH_KRY)))
      continue;
    const typename SP::W w = SP::ws(b, slot);
    double yv[N], fv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) yv[k] = w.yq(k);
    int rv;
    if constexpr (V::SM) {
      extern __shared__ double rsm[];   // 2K doubles per thread, column-major by thread
      rv = Mech::template rhs_sm<V::BLOCK>(yv, t->aux, fv, rsm + threadIdx.x);
    } else {
      rv = Mech::rhs(yv, t->aux, fv);
    }
    if constexpr (LS == LS_DENSE && BDFB_SPLIT_RHS_SOLVE && N <= 32) {
      if (rv == 0 && ph == PH_NRES && !t->setup) {
        // consume (PH_NRES: del = -gamma f + (rl1 zn[1] + ycor)) and SOLVE (LU_SOLVE on the slot's record, the
        // stale-gamma scaling) of TpcIntegrator / Split::solve, operation for operation
        const double rl1 = t->rl1, gm = t->gamma, gamrat = t->gamrat;
        const double* lu = SP::lurec(b, slot);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double fr = fv[i] + w.fext(i);
          const double tt = rl1 * w.zn(1, i) + w.acor(i);
          w.del(i) = -gm * fr + tt;
        }
        double x[N];
#pragma unroll
        for (int i = 0; i < N; ++i) x[i] = -w.del(SP::lu_perm(lu, i));
        lurec_substitute<N, LU_STRIDE>(lu, x);
        if (gamrat != 1.0) {
          const double sc = 2.0 / (1.0 + gamrat);
#pragma unroll
          for (int i = 0; i < N; ++i) x[i] = sc * x[i];
        }
#pragma unroll
        for (int i = 0; i < N; ++i) w.del(i) = x[i];
        b.rv[slot] = RV_SOLVED;
        continue;
      }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) w.fr(k) = fv[k] + w.fext(k);
    b.rv[slot] = rv;
  }
}

}  // namespace bdfb
