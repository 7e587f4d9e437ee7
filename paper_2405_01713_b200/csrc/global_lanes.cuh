// global_lanes.cuh -- device kernels of the global-norm mode (row a12, the
// paper's lockstep batch) for mechanisms of any size n <= 64 (config
// C5: 53 species + T, n = 54), built on the table-driven group model
// ModelMechR (mech_lanes.cuh: one cell per group of G lanes, lane l owning
// components l + G r).  The generated straight-line thread-per-cell code
// (global_tpc.cuh) does not scale to a 325-reaction mechanism (compile time),
// so here:
//   gl_rhs:    f = R(y) + F, one cell per warp (table-driven RHS);
//   gl_setup:  [J = dR/dy, the analytic Jacobian, into HBM]; M = I - gamma J
//              in shared memory; LU with partial pivoting by the warp
//              (glu_factor_r: lane-owned rows, LAPACK position tracking,
//              reciprocal-multiply column scaling and fma updates -- the
//              listing's LU_FACTOR operation for operation, reading R16);
//              factors written in pivoted row order (row-major by position,
//              cell-minor: element e of cell c at [e N + c]) with perm[] and
//              1/U_kk, the layout of tpc_solve;
//   gl_solve:  b = M^{-1}(-del) (tpc_solve = LU_SOLVE), the stale-gamma scale,
//              acor += b, tmp = b (thread per cell, coalesced).
// Every other kernel of the mode (vectors, deterministic norms, the NCCL rank
// exchange) is shared with the other mechanisms (global_mode.cuh).
#pragma once
#include <utility>
#include "bdf_tpc.cuh"
#include "mech_lanes.cuh"

namespace bdfb {

// LU with partial pivoting of the n x n matrix A (shared, column-major with odd stride MS: A[j MS + i]) by a group
// of G lanes owning rows i = lane + G r.  Rows never move; pos[r] is row i's LAPACK position.  Per column k: the
// first position (ties: smaller position) of max |a_ik| over positions >= k by a group butterfly, r = 1/pivot once,
// multipliers m = a_ik r, a_ij = fma(-m, a_pj, a_ij).  Returns 0 or k+1 for an exact zero pivot (group-uniform).
// dinv[r] = 1/U at the row's position.
template <int N, int G, int MS>
__device__ int glu_factor_r(const Grp<G>& g, double* A, int (&pos)[(N + G - 1) / G], double (&dinv)[(N + G - 1) / G]) {
  constexpr int R = (N + G - 1) / G;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    pos[r] = g.lane + G * r;
    dinv[r] = 0.0;
  }
  for (int k = 0; k < N; ++k) {
    double bv = -1.0;
    int bp = 0x7fffffff, br = -1;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = g.lane + G * r;
      if (i < N && pos[r] >= k) {
        const double v = fabs(A[k * MS + i]);
        if (v > bv || (v == bv && pos[r] < bp)) {
          bv = v;
          bp = pos[r];
          br = i;
        }
      }
    }
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) {
      const double ov = __shfl_xor_sync(g.mask, bv, off, G);
      const int op = __shfl_xor_sync(g.mask, bp, off, G);
      const int orr = __shfl_xor_sync(g.mask, br, off, G);
      if (ov > bv || (ov == bv && op < bp)) {
        bv = ov;
        bp = op;
        br = orr;
      }
    }
    if (!(bv > 0.0)) {
      g.sync();
      return k + 1;
    }
    const double pv = A[k * MS + br];
    const double rinv = 1.0 / pv;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = g.lane + G * r;
      if (i == br) {
        pos[r] = k;
        dinv[r] = rinv;
      } else if (i < N && pos[r] == k) {
        pos[r] = bp;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = g.lane + G * r;
      if (i < N && pos[r] > k) {
        const double m = A[k * MS + i] * rinv;
        A[k * MS + i] = m;
        for (int j = k + 1; j < N; ++j) A[j * MS + i] = fma(-m, A[j * MS + br], A[j * MS + i]);
      }
    }
    g.sync();
  }
  return 0;
}

template <class MR>
struct GLK {
  static constexpr int NN = MR::N, G = MR::G, R = MR::R;
  static constexpr int MS = NN | 1;
  static constexpr int PG_RHS = MR::SG;                        // shared doubles per group, gl_rhs
  static constexpr int PG_SET = NN * MS + MR::SG + MR::JG;     // shared doubles per group, gl_setup
  static constexpr int GPB = 128 / G;                          // groups per 128-thread block
};

template <class MR>
__global__ void __launch_bounds__(128) gl_rhs(long long N, const double* y, const double* fext, const double* aux,
                                              double* f, int* flag) {
  using K = GLK<MR>;
  constexpr int G = MR::G, NN = MR::N, R = MR::R;
  extern __shared__ double smem[];
  Grp<G> g;
  double* sc = smem + (threadIdx.x / G) * K::PG_RHS;
  const long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool live = grp < N;
  const long long c = live ? grp : 0;
  double yy[R], ff[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = g.lane + G * r;
    yy[r] = i < NN ? y[(long long)i * N + c] : 0.0;
  }
  const int rv = MR::rhs(g, yy, aux ? aux[c] : 0.0, ff, sc);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = g.lane + G * r;
    if (live && i < NN) f[(long long)i * N + c] = ff[r] + (fext ? fext[(long long)i * N + c] : 0.0);
  }
  if (live && rv && g.lane == 0) atomicOr(flag, 1);
}

// setup of one cell per group: (jbad) J at y into HBM; unless jac_only: M = I - gamma J; LU; factors + perm +
// 1/U to HBM.  (The default path calls it with jac_only = 1 and factors with gl_lu.)
template <class MR>
__global__ void __launch_bounds__(128) gl_setup(long long N, int jbad, double gamma, const double* y,
                                                const double* aux, double* J, double* LU, int* perm, double* invd,
                                                int* flag, int jac_only) {
  using K = GLK<MR>;
  constexpr int G = MR::G, NN = MR::N, R = MR::R, MS = K::MS;
  extern __shared__ double smem[];
  Grp<G> g;
  double* A = smem + (threadIdx.x / G) * K::PG_SET;
  double* sc = A + NN * MS;
  double* js = sc + MR::SG;
  const long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool live = grp < N;
  const long long c = live ? grp : 0;
  int bad = 0;
  if (jbad) {
    double yy[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = g.lane + G * r;
      yy[r] = i < NN ? y[(long long)i * N + c] : 0.0;
    }
    bad = MR::jac(g, yy, aux ? aux[c] : 0.0, A, 1, MS, sc, js);   // row i, column j at A[j MS + i]
    if (live && !bad) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = g.lane + G * r;
        if (i < NN)
          for (int j = 0; j < NN; ++j) J[((long long)i * NN + j) * N + c] = A[j * MS + i];
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = g.lane + G * r;
      if (i < NN)
        for (int j = 0; j < NN; ++j) A[j * MS + i] = J[((long long)i * NN + j) * N + c];
    }
  }
  g.sync();
  if (!bad && !jac_only) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = g.lane + G * r;
      if (i < NN)
        for (int j = 0; j < NN; ++j) A[j * MS + i] = (i == j ? 1.0 : 0.0) - gamma * A[j * MS + i];
    }
    g.sync();
    int pos[R];
    double dinv[R];
    bad = glu_factor_r<NN, G, MS>(g, A, pos, dinv);
    if (live && !bad) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = g.lane + G * r;
        if (i < NN) {
          const long long p = pos[r];
          for (int j = 0; j < NN; ++j) LU[(p * NN + j) * N + c] = A[j * MS + i];
          perm[p * N + c] = i;
          invd[p * N + c] = dinv[r];
        }
      }
    }
  }
  if (live && bad && g.lane == 0) atomicOr(flag, 1);
}

// M = I - gamma J and its LU with partial pivoting, ONE CELL PER BLOCK of 32 ceil(n/32) threads, thread i
// owning row i of M in registers for the whole factorisation (columns fully unrolled).  Per column k: the
// pivot (max |m_ik| over rows at LAPACK positions >= k, ties to the smaller position) by a warp butterfly and
// an ordered combination of the warps' candidates in shared memory; the pivot row's owner publishes its row
// and 1/pivot; every row below forms its multiplier m = m_ik (1/pivot) and applies fma(-m, u_kj, m_ij) --
// the listing's LU_FACTOR operation for operation (reading R16), as glu_factor_r, so factors and pivots are
// bit-identical.  Versus the shared-memory warp LU of gl_setup (3 shared-memory accesses per FMA, 8 warps per
// SM): the update is one broadcast shared load per FMA from registers, 16 warps per SM.  Factors written in
// pivoted row order, cell-minor (element e of cell c at [e N + c]) with perm and 1/U_kk (tpc_solve layout).
// CPB cells per block of CPB x 32 ceil(n/32) threads: all 12 warps of an SM walk the same column of the
// unrolled factorisation together (one barrier pair per column for all six cells: instruction-cache locality)
template <int NN>
#ifndef BDFB_GLU_THREADS
#define BDFB_GLU_THREADS 384   // threads per block; 384 / BDFB_GLU_THREADS blocks per SM (the 12 warps either way)
#endif
struct GLU {
  static constexpr int W = (NN + 31) / 32, TC = 32 * W,
                       CPB = BDFB_GLU_THREADS / TC > 0 ? BDFB_GLU_THREADS / TC : 1, T = CPB * TC,
                       BPS = 384 / T > 0 ? 384 / T : 1;   // resident blocks per SM
};
// shared state of a gl_lu block: per cell the published pivot row and 1/pivot, the warps' pivot candidates
// (double-buffered by column parity)
template <int NN>
struct GLUShared {
  double2 prow[2][GLU<NN>::CPB][NN / 2 + 1];
  double crv[2][GLU<NN>::CPB][GLU<NN>::W], srinv[2][GLU<NN>::CPB];
  int crp[2][GLU<NN>::CPB][GLU<NN>::W], crr[2][GLU<NN>::CPB][GLU<NN>::W];
};
// column K of gl_lu (K a compile-time constant, so that the row stays in registers); returns false at an exact
// zero pivot (uniform per cell; the block keeps meeting the barriers)
template <int NN, int K>
__device__ __forceinline__ bool glu_column(GLUShared<NN>& sh, double (&a)[NN], int& pos, double& dinv, int i,
                                           int cb, bool alive) {
  constexpr int W = GLU<NN>::W, par = K & 1, J0 = (K + 1) & ~1;
  const int lane = i & 31, warp = i >> 5;
  const bool own = i < NN && alive;
  double bv = -1.0;
  int bp = 0x7fffffff, br = -1;
  if (own && pos >= K) {
    bv = fabs(a[K]);
    bp = pos;
    br = i;
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int op = __shfl_xor_sync(0xffffffffu, bp, off);
    const int orr = __shfl_xor_sync(0xffffffffu, br, off);
    if (ov > bv || (ov == bv && op < bp)) {
      bv = ov;
      bp = op;
      br = orr;
    }
  }
  if (lane == 0) {
    sh.crv[par][cb][warp] = bv;
    sh.crp[par][cb][warp] = bp;
    sh.crr[par][cb][warp] = br;
  }
  __syncthreads();
  bv = sh.crv[par][cb][0];
  bp = sh.crp[par][cb][0];
  br = sh.crr[par][cb][0];
#pragma unroll
  for (int w = 1; w < W; ++w) {
    const double ov = sh.crv[par][cb][w];
    const int op = sh.crp[par][cb][w];
    if (ov > bv || (ov == bv && op < bp)) {
      bv = ov;
      bp = op;
      br = sh.crr[par][cb][w];
    }
  }
  const bool ok = bv > 0.0;
  if (ok && i == br) {
    const double rinv = 1.0 / a[K];
    sh.srinv[par][cb] = rinv;
#pragma unroll
    for (int j = J0; j < NN; j += 2) sh.prow[par][cb][j / 2] = make_double2(a[j], j + 1 < NN ? a[j + 1] : 0.0);
    pos = K;
    dinv = rinv;
  } else if (ok && own && pos == K) {
    pos = bp;
  }
  __syncthreads();
  if (ok && own && pos > K) {
    const double m = a[K] * sh.srinv[par][cb];
    a[K] = m;
#pragma unroll
    for (int j = J0; j < NN; j += 2) {
      const double2 u = sh.prow[par][cb][j / 2];
      if (j > K) a[j] = fma(-m, u.x, a[j]);
      if (j + 1 < NN) a[j + 1] = fma(-m, u.y, a[j + 1]);
    }
  }
  return ok;
}
template <int NN, int... Ks>
__device__ __forceinline__ int glu_columns(GLUShared<NN>& sh, double (&a)[NN], int& pos, double& dinv, int i, int cb,
                                           bool alive, std::integer_sequence<int, Ks...>) {
  int info = 0;
  // every thread runs every column (block-wide barriers); a cell whose pivot was exactly zero stops updating
  (void)((glu_column<NN, Ks>(sh, a, pos, dinv, i, cb, alive && !info) || !alive || info || (info = Ks + 1, true)) &&
         ...);
  return info;
}

// M = I - gamma J and its LU with partial pivoting, one cell per 32 ceil(n/32) threads (CPB cells per block),
// thread i owning row i of M in registers for the whole factorisation (columns unrolled at compile time).  Per
// column k: the pivot (max |m_ik| over rows at LAPACK positions >= k, ties to the smaller position) by a warp
// butterfly and an ordered combination of the warps' candidates in shared memory; the pivot row's owner
// publishes its row and 1/pivot; every row below forms its multiplier m = m_ik (1/pivot) and applies
// fma(-m, u_kj, m_ij) -- the listing's LU_FACTOR operation for operation (reading R16), as glu_factor_r, so
// factors and pivots are bit-identical.  Versus the shared-memory warp LU of gl_setup (three shared-memory
// accesses per FMA, 8 warps per SM): one broadcast 16-byte shared load per two FMAs on register rows, 12 warps
// per SM in lockstep.  Factors written in pivoted row order, cell-minor (element e of cell c at [e N + c]) with
// perm and 1/U_kk (the tpc_solve layout).
template <int NN>
__global__ void __launch_bounds__(GLU<NN>::T, GLU<NN>::BPS)
    gl_lu(long long N, double gamma, const double* J, double* LU, int* perm, double* invd, int* flag) {
  __shared__ GLUShared<NN> sh;
  // the block's six matrices staged element-major, cell-minor (T[e CPB + cb]): the cell-minor HBM layout is then
  // read and written as runs of CPB consecutive cells instead of one scattered 8-byte access per row and column
  // (ncu: the scattered stores and loads were ~40% of the kernel's stall samples)
  extern __shared__ double T[];
  constexpr int TC = GLU<NN>::TC, CPB = GLU<NN>::CPB, E = NN * NN;
  const int cb = threadIdx.x / TC, i = threadIdx.x % TC;
  const long long c0 = (long long)blockIdx.x * CPB, c = c0 + cb;
  const int ncb = N - c0 < CPB ? (int)(N - c0) : CPB;
  for (int x = threadIdx.x; x < E * CPB; x += blockDim.x) {
    const int e = x / CPB, cc = x - e * CPB;
    if (cc < ncb) T[x] = J[(long long)e * N + c0 + cc];
  }
  __syncthreads();
  const bool alive = c < N;
  const bool own = i < NN && alive;
  double a[NN];
#pragma unroll
  for (int j = 0; j < NN; ++j) a[j] = own ? (i == j ? 1.0 : 0.0) - gamma * T[(i * NN + j) * CPB + cb] : 0.0;
  int pos = i;
  double dinv = 0.0;
  const int info = glu_columns<NN>(sh, a, pos, dinv, i, cb, alive, std::make_integer_sequence<int, NN>{});
  if (alive && info && i == 0) atomicOr(flag, 1);
  if (own && !info) {
    const int p = pos;
#pragma unroll
    for (int j = 0; j < NN; ++j) T[(p * NN + j) * CPB + cb] = a[j];
    perm[(long long)p * N + c] = i;
    invd[(long long)p * N + c] = dinv;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < E * CPB; x += blockDim.x) {
    const int e = x / CPB, cc = x - e * CPB;
    if (cc < ncb) LU[(long long)e * N + c0 + cc] = T[x];
  }
}

template <int NN>
constexpr size_t gl_lu_smem() {
  return sizeof(double) * (size_t)NN * NN * GLU<NN>::CPB;
}

template <int NN>
__global__ void __launch_bounds__(128) gl_solve(long long N, double sc2, const double* LU, const int* perm,
                                                const double* invd, const double* del, double* acor, double* tmp) {
  const long long c = (long long)blockIdx.x * 128 + threadIdx.x;
  if (c >= N) return;
  double x[NN];
  tpc_solve<NN, true, 0>(LU + c, invd + c, perm + c, del + c, N, x);
#pragma unroll
  for (int k = 0; k < NN; ++k) {
    const double b = (sc2 != 1.0) ? sc2 * x[k] : x[k];
    const long long e = (long long)k * N + c;
    acor[e] = acor[e] + b;
    tmp[e] = b;
  }
}

}  // namespace bdfb
