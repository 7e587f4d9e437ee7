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

// setup of one cell per group: (jbad) J at y into HBM; M = I - gamma J; LU; factors + perm + 1/U to HBM
template <class MR>
__global__ void __launch_bounds__(128) gl_setup(long long N, int jbad, double gamma, const double* y,
                                                const double* aux, double* J, double* LU, int* perm, double* invd,
                                                int* flag) {
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
  if (!bad) {
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
