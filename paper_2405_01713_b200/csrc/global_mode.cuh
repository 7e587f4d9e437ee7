// global_mode.cuh -- the paper's lockstep batch ("global-norm mode", §8 row
// a12; listing "Global-norm variant"; reading R14).
//
// All cells of all ranks form ONE system of n * N_total components: one h,
// q and Nordsieck history; every WRMS norm is batch-wide with N = n * N_total;
// the Jacobian is block diagonal (one n x n LU per cell, HBM-resident); any
// cell's zero pivot or RHS failure is the batch's recoverable failure (R18).
//
// Execution model = the paper's: the integrator's scalar logic runs on the
// host, the vector operations run as device kernels over all cells.
// Each norm is a deterministic reduction: per-cell sums (components in
// increasing order), block partials over ORC-equivalent blocks of 256 cells in
// cell order, then the block partials in order, then (multi-rank) the rank
// partials in rank order after an ncclAllGather -- so every rank takes the
// same decisions and the result matches the oracle's specified order (R15).
//
// Device layout: vectors YC (k*N + c), J and LU cell-major (c*n*n + i*n + j).
#pragma once
#include "bdf_group.cuh"

namespace bdfb {

constexpr int GM_BLK = 256;   // cells per partial sum (== oracle ORC_GBLK)

struct GVec {                 // device vectors of the global state (YC, n*N)
  double* zn[QMAX + 1];
  double *ewt, *acor, *yq, *fy, *del, *tmp, *f;
};

// ---- elementwise kernels: one thread per cell, components in order ----------
__global__ void gk_predict(GVec v, int n, long long N, int q) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= N) return;
  for (int i = 0; i < n; ++i) {
    const long long e = (long long)i * N + c;
    for (int k = 1; k <= q; ++k)
      for (int j = q; j >= k; --j) v.zn[j - 1][e] = v.zn[j - 1][e] + v.zn[j][e];
  }
}
__global__ void gk_restore(GVec v, int n, long long N, int q) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= N) return;
  for (int i = 0; i < n; ++i) {
    const long long e = (long long)i * N + c;
    for (int k = 1; k <= q; ++k)
      for (int j = q; j >= k; --j) v.zn[j - 1][e] = v.zn[j - 1][e] - v.zn[j][e];
  }
}
__global__ void gk_rescale(GVec v, int n, long long N, int q, double eta) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= N) return;
  for (int i = 0; i < n; ++i) {
    const long long e = (long long)i * N + c;
    double r = eta;
    for (int j = 1; j <= q; ++j) {
      v.zn[j][e] = r * v.zn[j][e];
      r = r * eta;
    }
  }
}
struct GCoef { double c[QMAX + 1]; };
// zn[j] = l[j] * acor + zn[j] (j <= q); optionally zn[qmax] = acor
__global__ void gk_complete(GVec v, int n, long long N, int q, GCoef l, int save, int qmax) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= N) return;
  for (int i = 0; i < n; ++i) {
    const long long e = (long long)i * N + c;
    const double a = v.acor[e];
    for (int j = 0; j <= q; ++j) v.zn[j][e] = l.c[j] * a + v.zn[j][e];
    if (save) v.zn[qmax][e] = a;
  }
}
// order increase: zn[q+1] = A1 zn[qmax]; zn[j] += lc[j] zn[q+1] (2 <= j <= q)
__global__ void gk_increase(GVec v, int n, long long N, int q, int qmax, double A1, GCoef lc) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= N) return;
  for (int i = 0; i < n; ++i) {
    const long long e = (long long)i * N + c;
    const double zL = A1 * v.zn[qmax][e];
    v.zn[q + 1][e] = zL;
    for (int j = 2; j <= q; ++j) v.zn[j][e] = lc.c[j] * zL + v.zn[j][e];
  }
}
// order decrease: zn[j] = -lc[j] zn[q] + zn[j] (2 <= j < q)
__global__ void gk_decrease(GVec v, int n, long long N, int q, GCoef lc) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= N) return;
  for (int i = 0; i < n; ++i) {
    const long long e = (long long)i * N + c;
    const double zq = v.zn[q][e];
    for (int j = 2; j < q; ++j) v.zn[j][e] = -lc.c[j] * zq + v.zn[j][e];
  }
}
// generic: dst = a * x + b * y (elementwise, all n*N)
__global__ void gk_axpby(double* dst, double a, const double* x, double b, const double* y, long long M) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= M) return;
  dst[e] = (y ? a * x[e] + b * y[e] : a * x[e]);
}
__global__ void gk_ewt(double* ewt, const double* y, const double* atol, double rtol, int n, long long N) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * N) return;
  ewt[e] = 1.0 / (rtol * fabs(y[e]) + atol[e / N]);
}
// residual: fy = f; del = -gamma f + (rl1 zn1 + acor)
__global__ void gk_residual(GVec v, long long M, double gamma, double rl1) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= M) return;
  const double f = v.f[e];
  v.fy[e] = f;
  const double t = rl1 * v.zn[1][e] + v.acor[e];
  v.del[e] = -gamma * f + t;
}
// per-cell sum of (w v)^2, components in increasing order (G = 1 order)
__global__ void gk_cellsum(const double* x, const double* w, double* s, int n, long long N) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= N) return;
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const double p = x[(long long)i * N + c] * w[(long long)i * N + c];
    acc = acc + p * p;
  }
  s[c] = acc;
}
// block partials: P[b] = sum over GM_BLK consecutive cells in order
__global__ void gk_blocksum(const double* s, double* P, long long N) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long c0 = b * GM_BLK;
  if (c0 >= N) return;
  const long long c1 = c0 + GM_BLK < N ? c0 + GM_BLK : N;
  double acc = 0.0;
  for (long long c = c0; c < c1; ++c) acc = acc + s[c];
  P[b] = acc;
}
// the block partials summed in order (reading R15: bit-reproducible); the block stages chunks of P in
// shared memory with coalesced loads so that the one sequential summing thread reads on-chip operands
constexpr int GK_FINAL_THREADS = 256, GK_FINAL_CHUNK = 4096;
__global__ void __launch_bounds__(GK_FINAL_THREADS) gk_finalsum(const double* P, long long nb, double* out) {
  __shared__ double sp[GK_FINAL_CHUNK];
  double acc = 0.0;
  for (long long b0 = 0; b0 < nb; b0 += GK_FINAL_CHUNK) {
    const int m = (int)(nb - b0 < GK_FINAL_CHUNK ? nb - b0 : GK_FINAL_CHUNK);
    for (int i = threadIdx.x; i < m; i += GK_FINAL_THREADS) sp[i] = P[b0 + i];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < m; ++i) acc = acc + sp[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = acc;
}
// max_i |zn1| / (0.1 |zn0| + 1/ewt)  (cvUpperBoundH0) -> atomicMax on the bits of a positive double
__global__ void gk_hubinv(GVec v, long long M, unsigned long long* out) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double r = 0.0;
  if (e < M) {
    const double d = HUB_FACTOR * fabs(v.zn[0][e]) + 1.0 / v.ewt[e];
    r = fabs(v.zn[1][e]) / d;
  }
  for (int off = 16; off >= 1; off >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(r));
}
__global__ void gk_finite(const double* x, long long M, int* flag) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < M && !isfinite(x[e])) atomicOr(flag, 1);
}

// ---- model kernels: one cell per group of G lanes ------------------------------
template <class Model>
struct GMK {
  static constexpr int N_ = Model::N, G = Model::G;
  static constexpr int MS = GroupIntegrator<Model>::MS;
  static constexpr int PG = N_ * MS + Model::SG + Model::JG + 2 * G + 2 * G;   // per group (doubles)
  static constexpr int GPB = 128 / G;                                         // groups per block
};

// f = R(t, y) + F for every cell; *flag |= 1 on any recoverable RHS failure
template <class Model>
__global__ void __launch_bounds__(128) gk_rhs(typename Model::Params prm, long long N, double t, const double* y,
                                              const double* fext, const double* aux, double* f, int* flag) {
  using K = GMK<Model>;
  constexpr int G = Model::G, NN = Model::N;
  extern __shared__ double smem[];
  Grp<G> g;
  const int gi = threadIdx.x / G;
  double* sc = smem + gi * K::PG + NN * K::MS;
  const long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool live = grp < N;
  const long long c = live ? grp : 0;
  double yy[1] = {g.lane < NN ? y[(long long)g.lane * N + c] : 0.0}, ff[1];
  const int rv = Model::rhs(g, prm, t, yy, ff, aux ? aux[c] : 0.0, sc);
  if (live && g.lane < NN) f[(long long)g.lane * N + c] = ff[0] + (fext ? fext[(long long)g.lane * N + c] : 0.0);
  if (live && rv && g.lane == 0) atomicOr(flag, 1);
}

// setup: (jbad: J = dR/dy at y) ; M = I - gamma J ; LU (positions, permutation, 1/U_kk)
template <class Model>
__global__ void __launch_bounds__(128) gk_setup(typename Model::Params prm, long long N, int jbad, double gamma,
                                                const double* y, const double* aux, double* J, double* LU,
                                                int* pos, int* perm, double* invd, int* flag) {
  using K = GMK<Model>;
  constexpr int G = Model::G, NN = Model::N, MS = K::MS;
  extern __shared__ double smem[];
  Grp<G> g;
  const int gi = threadIdx.x / G;
  double* A = smem + gi * K::PG;
  double* sc = A + NN * MS;
  double* js = sc + Model::SG;
  int* ip = reinterpret_cast<int*>(js + Model::JG);
  int* pp = ip + G;
  double* iv = reinterpret_cast<double*>(pp + G);
  const long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool live = grp < N;
  const long long c = live ? grp : 0;
  double* Jc = J + c * NN * NN;
  int bad = 0;
  if (jbad) {
    bad = Model::template jac<MS>(g, g.lane < NN ? y[(long long)g.lane * N + c] : 0.0, aux ? aux[c] : 0.0,
                                  A + g.lane, sc, js);
    if (live && g.lane < NN)
      for (int j = 0; j < NN; ++j) Jc[g.lane * NN + j] = A[j * MS + g.lane];
    g.sync();
  }
  if (!bad) {
    if (g.lane < NN)
      for (int j = 0; j < NN; ++j) A[j * MS + g.lane] = (g.lane == j ? 1.0 : 0.0) - gamma * Jc[g.lane * NN + j];
    g.sync();
    bad = glu_factor<NN, G, MS>(g, A, ip, pp, iv);
  }
  if (live) {
    if (g.lane < NN && !bad) {
      for (int j = 0; j < NN; ++j) LU[c * NN * NN + g.lane * NN + j] = A[j * MS + g.lane];
      pos[c * NN + g.lane] = ip[g.lane];
      perm[c * NN + g.lane] = pp[g.lane];
      invd[c * NN + g.lane] = iv[g.lane];
    }
    if (bad && g.lane == 0) atomicOr(flag, 1);
  }
}

// b = M^{-1} (-del) (x 2/(1+gamrat) if gamrat != 1); acor += b; tmp = b
template <class Model>
__global__ void __launch_bounds__(128) gk_solve(long long N, double sc2, const double* LU, const int* pos,
                                                const int* perm, const double* invd, const double* del, double* acor,
                                                double* tmp) {
  using K = GMK<Model>;
  constexpr int G = Model::G, NN = Model::N, MS = K::MS;
  extern __shared__ double smem[];
  Grp<G> g;
  const int gi = threadIdx.x / G;
  double* A = smem + gi * K::PG;
  int* pp = reinterpret_cast<int*>(A + NN * MS);
  const long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool live = grp < N;
  const long long c = live ? grp : 0;
  if (g.lane < NN) {
    for (int j = 0; j < NN; ++j) A[j * MS + g.lane] = LU[c * NN * NN + g.lane * NN + j];
    pp[g.lane] = perm[c * NN + g.lane];
  }
  g.sync();
  const int p = g.lane < NN ? pos[c * NN + g.lane] : g.lane;
  const double iv = g.lane < NN ? invd[c * NN + g.lane] : 0.0;
  double b = g.lane < NN ? -del[(long long)g.lane * N + c] : 0.0;
  b = glu_solve<NN, G, MS>(g, A, p, iv, pp, b);
  if (sc2 != 1.0) b = sc2 * b;
  if (live && g.lane < NN) {
    const long long e = (long long)g.lane * N + c;
    acor[e] = acor[e] + b;
    tmp[e] = b;
  }
}

}  // namespace bdfb
