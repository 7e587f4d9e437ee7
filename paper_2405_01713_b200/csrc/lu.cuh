// lu.cuh -- in-group dense LU with partial pivoting and solve, fp64, no
// tensor cores (the per-cell systems are n <= 32: not a dense contraction).
//
// Operation semantics are the listing's LU_FACTOR / LU_SOLVE (SURVEY.md
// §8(c).2, reading R16; "LU factorization with pivoting"):
//   pivot = first index of max |M[i][k]| over the not-yet-pivoted rows,
//   exact zero pivot -> singular (recoverable), reciprocal-multiply column
//   scaling, fma updates, axpy-ordered substitutions.
//
// Storage: the matrix of a warp lives in shared memory, element (row i, col
// j) of a group at  A[(slot*N + j)*WS + warp_lane]  where row i is owned by
// group lane (i mod G) in register slot i / G.  WS = 33 pads the lane stride
// so that row-parallel and broadcast accesses are bank-conflict free.
//
// G > 1 (one row per lane, N <= G): rows never move between lanes.  Each lane
// tracks the position `pos` its row would occupy in LAPACK's physically
// swapped factor; the pivot search breaks ties by smallest position exactly
// as LAPACK's first-max does, so pivots and factors are bit-identical to the
// listing.  perm[k] = lane holding position k (group-local smem).
// G = 1 (one thread owns all N rows): the listing with physical row swaps.
#pragma once
#include "grp.cuh"

namespace bdfb {

constexpr int WS = 33;  // padded warp stride of matrix storage (doubles)

template <int N, int G>
__device__ __forceinline__ double& mat(double* A, const Grp<G>& g, int slot, int j) {
  return A[(slot * N + j) * WS + g.wlane];
}

// ---- G > 1 ------------------------------------------------------------------
template <int N, int G>
__device__ int lu_factor_group(const Grp<G>& g, double* A, int& pos, int* perm) {
  static_assert(G > 1 && N <= G, "one row per lane");
  const bool act = g.lane < N;
  pos = g.lane;
  for (int k = 0; k < N; ++k) {
    double a = (act && pos >= k) ? fabs(A[k * WS + g.wlane]) : -1.0;
    int key = (pos << 5) | g.lane;
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) {
      double oa = __shfl_xor_sync(g.mask, a, off, G);
      int ok = __shfl_xor_sync(g.mask, key, off, G);
      if (oa > a || (oa == a && ok < key)) { a = oa; key = ok; }
    }
    const int p = key >> 5, pl = key & 31;
    const double pv = A[k * WS + g.gbase + pl];
    if (pv == 0.0) { g.sync(); return k + 1; }
    if (g.lane == pl) pos = k;
    else if (pos == k) pos = p;
    if (act && pos > k) {
      const double r = 1.0 / pv;
      const double m = A[k * WS + g.wlane] * r;
      A[k * WS + g.wlane] = m;
      for (int j = k + 1; j < N; ++j)
        A[j * WS + g.wlane] = fma(-m, A[j * WS + g.gbase + pl], A[j * WS + g.wlane]);
    }
    g.sync();
  }
  if (act) perm[g.gbase + pos] = g.lane;
  g.sync();
  return 0;
}

// reciprocal of this lane's U diagonal (its row's entry in column pos);
// reading R16: the solve multiplies by 1/U[k][k] instead of dividing.
template <int N, int G>
__device__ __forceinline__ double lu_inv_diag(const Grp<G>& g, const double* A, int pos) {
  return (g.lane < N) ? 1.0 / A[pos * WS + g.wlane] : 0.0;
}

// b: this lane's right-hand-side component (row = lane); returns x[lane].
// perm[] is read once into registers (the loops are unrolled).
template <int N, int G>
__device__ double lu_solve_group(const Grp<G>& g, const double* A, int pos, double invd, const int* perm, double b) {
  const bool act = g.lane < N;
  int src[N];
#pragma unroll
  for (int k = 0; k < N; ++k) src[k] = perm[g.gbase + k];
#pragma unroll
  for (int k = 0; k < N - 1; ++k) {
    const double bk = __shfl_sync(g.mask, b, src[k], G);
    if (act && pos > k) b = fma(-A[k * WS + g.wlane], bk, b);
  }
#pragma unroll
  for (int k = N - 1; k > 0; --k) {
    if (act && pos == k) b = b * invd;
    const double bk = __shfl_sync(g.mask, b, src[k], G);
    if (act && pos < k) b = fma(-A[k * WS + g.wlane], bk, b);
  }
  if (act && pos == 0) b = b * invd;
  const int from = act ? perm[g.gbase + g.lane] : g.lane;
  return __shfl_sync(g.mask, b, from, G);
}

// ---- G = 1 ------------------------------------------------------------------
template <int N>
__device__ int lu_factor_thread(const Grp<1>& g, double* A, int (&piv)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int p = k;
    double amax = fabs(mat<N, 1>(A, g, k, k));
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      double a = fabs(mat<N, 1>(A, g, i, k));
      if (a > amax) { amax = a; p = i; }
    }
    piv[k] = p;
    if (A[(p * N + k) * WS + g.wlane] == 0.0) return k + 1;
    if (p != k) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double t = mat<N, 1>(A, g, k, j);
        mat<N, 1>(A, g, k, j) = A[(p * N + j) * WS + g.wlane];
        A[(p * N + j) * WS + g.wlane] = t;
      }
    }
    const double r = 1.0 / mat<N, 1>(A, g, k, k);
#pragma unroll
    for (int i = k + 1; i < N; ++i) mat<N, 1>(A, g, i, k) *= r;
#pragma unroll
    for (int i = k + 1; i < N; ++i)
#pragma unroll
      for (int j = k + 1; j < N; ++j)
        mat<N, 1>(A, g, i, j) = fma(-mat<N, 1>(A, g, i, k), mat<N, 1>(A, g, k, j), mat<N, 1>(A, g, i, j));
  }
  return 0;
}

template <int N>
__device__ void lu_solve_thread(const Grp<1>& g, const double* A, const int (&piv)[N], double (&b)[N]) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const int p = piv[k];
#pragma unroll
    for (int i = k + 1; i < N; ++i)
      if (i == p) { double t = b[k]; b[k] = b[i]; b[i] = t; }
  }
#pragma unroll
  for (int k = 0; k < N - 1; ++k)
#pragma unroll
    for (int i = k + 1; i < N; ++i) b[i] = fma(-A[(i * N + k) * WS + g.wlane], b[k], b[i]);
#pragma unroll
  for (int k = N - 1; k > 0; --k) {
    b[k] = b[k] * (1.0 / A[(k * N + k) * WS + g.wlane]);
#pragma unroll
    for (int i = 0; i < k; ++i) b[i] = fma(-A[(i * N + k) * WS + g.wlane], b[k], b[i]);
  }
  b[0] = b[0] * (1.0 / A[g.wlane]);
}

}  // namespace bdfb
