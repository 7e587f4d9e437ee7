// split.cu -- the SPLIT per-cell integrator (bdf_split.cuh): slot pool
// geometry, the five kernels of a trip and the host loop that enqueues them;
// a translation unit of libbdfb.so, used by bdfb.cu through split_api.h.
#include <cuda_runtime.h>
#include <stdlib.h>

#include "../../include/bdfb.h"
#include "bdf_split.cuh"
#include "gen/mech_drm19_class.cuh"
#include "gen/mech_h2_lidryer.cuh"
#include "gen/tpc_drm19_class.cuh"
#include "gen/tpc_h2_lidryer.cuh"
#include "mech_model.cuh"
#include "split_api.h"
#include "split_run.cuh"

namespace bdfb {
namespace {

// LU diagnostic: the SPLIT path's own factor/solve routines on identical inputs
// (oct_factor, 8 lanes per cell, as K_lu; the record layout of K_lu; the
// thread-level substitutions of K_ctl's Newton solve, lurec_substitute).
// M[(i n + j) N + c] in, LAPACK getrf factors out (rows in pivoted order);
// piv: getrf swap indices derived from the row permutation; b: solution.
template <int NN>
__global__ void __launch_bounds__(128) split_lu_diag_kernel(long long N, double* M, int* piv, double* b, int* info,
                                                            double* rec) {
  constexpr int R = (NN + OCT - 1) / OCT;
  constexpr int S = LU_STRIDE;
  constexpr int LUREC = S == 1 ? (NN * NN + NN + (NN + 1) / 2 + 3) / 4 * 4 : NN * NN + 2 * NN;
  constexpr int LU_INVD = NN * NN, LU_PERM = NN * NN + NN;
  const int lane = threadIdx.x & 31, gl = lane & (OCT - 1);
  const long long c = ((long long)blockIdx.x * 128 + threadIdx.x) / OCT;
  const bool have = c < N;                    // the whole warp factors (oct_factor is warp-collective)
  if (__all_sync(0xffffffffu, !have)) return;
  double* lu = S == 1 ? rec + c * LUREC : rec + ((c >> 5) * LUREC) * 32 + (c & 31);   // K_lu's record layout
  double a[R][NN];
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int r = gl + OCT * s;
#pragma unroll
    for (int j = 0; j < NN; ++j) a[s][j] = (r < NN) ? (have ? M[((long long)r * NN + j) * N + c] : (r == j ? 1.0 : 0.0)) : 0.0;
  }
  int pos[R];
  double dinv[R];
  const int inf = oct_factor<NN>(gl, a, pos, dinv);
  if (!have) return;
  if (!inf) {
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int r = gl + OCT * s;
      if (r < NN) {
#pragma unroll
        for (int j = 0; j < NN; ++j) lu[(j * NN + pos[s]) * S] = a[s][j];
        lu[(LU_INVD + pos[s]) * S] = dinv[s];
        if (S == 1) reinterpret_cast<int*>(lu + LU_PERM)[pos[s]] = r;
        else lu[(LU_PERM + pos[s]) * S] = (double)r;
      }
    }
  }
  __syncwarp(__activemask());
  if (gl != 0) return;
  info[c] = inf;
  if (inf) return;
  int perm[NN];
#pragma unroll
  for (int i = 0; i < NN; ++i)
    perm[i] = S == 1 ? reinterpret_cast<const int*>(lu + LU_PERM)[i] : (int)lu[(LU_PERM + i) * S];
  double x[NN];
#pragma unroll
  for (int i = 0; i < NN; ++i) x[i] = b[(long long)perm[i] * N + c];
  lurec_substitute<NN, S>(lu, x);
  for (int i = 0; i < NN; ++i) {
    b[(long long)i * N + c] = x[i];
    for (int j = 0; j < NN; ++j) M[((long long)i * NN + j) * N + c] = lu[(j * NN + i) * S];
  }
  // getrf swap sequence of the permutation: at step k the row perm[k] sits at position where[perm[k]]
  int cur[NN], where[NN];
  for (int i = 0; i < NN; ++i) cur[i] = where[i] = i;
  for (int k = 0; k < NN; ++k) {
    const int p = where[perm[k]];
    piv[(long long)k * N + c] = p;
    const int rk = cur[k], rp = cur[p];
    cur[k] = rp;
    cur[p] = rk;
    where[rp] = k;
    where[rk] = p;
  }
}

// Jacobian diagnostic: the SPLIT path's two-pass generated Jacobian (jac_part / jac_sum / jac_col, the device
// functions of split_jac_part/sum/p2_kernel, the same warp-uniform part and column mapping and the same
// warp-blocked scratch) on N states in YC layout; J[(i n + j) N + c] out.
template <class Mech>
__global__ void __launch_bounds__(128) jd_pack(long long N, long long Nst, long long c0, const double* y, double* yb) {
  constexpr int n = Mech::N;
  const long long c = blockIdx.x * 128ll + threadIdx.x;
  if (c >= N) return;
  for (int k = 0; k < n; ++k) yb[((c >> 5) * n + k) * 32 + (c & 31)] = y[(long long)k * Nst + c0 + c];
}
template <class Mech>
__global__ void __launch_bounds__(128) jd_part(long long N, const double* yb, const double* aux, double* scr,
                                               int* status) {
  constexpr int n = Mech::N;
  const long long neb = (N + 31) / 32, nw = neb * Mech::NPART;
  const int lane = threadIdx.x & 31;
  for (long long gw = (blockIdx.x * 128ll + threadIdx.x) >> 5; gw < nw; gw += (gridDim.x * 128ll) >> 5) {
    const int P = (int)(gw / neb);
    const long long e = (gw - P * neb) * 32 + lane;
    if (e >= N) continue;
    const int rv = Mech::template jac_part<32, 32>(P, yb + ((e >> 5) * n) * 32 + (e & 31), aux[e],
                                                   scr + ((e >> 5) * Mech::NSC3) * 32 + (e & 31));
    if (P == 0) status[e] = rv;
  }
}
template <class Mech>
__global__ void __launch_bounds__(128) jd_sum(long long N, const double* yb, const double* aux, double* scr,
                                              const int* status) {
  constexpr int n = Mech::N;
  const long long e = blockIdx.x * 128ll + threadIdx.x;
  if (e >= N || status[e]) return;
  Mech::template jac_sum<32, 32>(yb + ((e >> 5) * n) * 32 + (e & 31), aux[e],
                                 scr + ((e >> 5) * Mech::NSC3) * 32 + (e & 31));
}
template <class Mech>
__global__ void __launch_bounds__(128) jd_col(long long N, const double* scr, const int* status, double* Jrec) {
  constexpr int n = Mech::N;
  const long long neb = (N + 31) / 32, nw = neb * n;
  const int lane = threadIdx.x & 31;
  for (long long gw = (blockIdx.x * 128ll + threadIdx.x) >> 5; gw < nw; gw += (gridDim.x * 128ll) >> 5) {
    const int j = (int)(gw / neb);
    const long long e = (gw - j * neb) * 32 + lane;
    if (e >= N || status[e]) continue;
    Mech::template jac_col<32>(j, scr + ((e >> 5) * Mech::NSC3) * 32 + (e & 31), Jrec + e * (n * n));
  }
}
template <class Mech>
__global__ void __launch_bounds__(128) jd_unpack(long long N, long long Nst, long long c0, const double* Jrec,
                                                 const int* status, double* J, int* flag) {
  constexpr int n = Mech::N;
  const long long c = blockIdx.x * 128ll + threadIdx.x;
  if (c >= N) return;
  if (status[c]) {
    if (flag) atomicOr(flag, 1);
    return;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) J[((long long)i * n + j) * Nst + c0 + c] = Jrec[c * (n * n) + j * n + i];
}
// N cells in chunks of at most JD_CHUNK (one scratch allocation): y[k N + c] in, J[(i n + j) N + c] out
constexpr long long JD_CHUNK = 65536;
template <class Mech>
cudaError_t jac_diag(long long N, const double* y, const double* aux, double* J, int* flag, cudaStream_t st) {
  constexpr int n = Mech::N;
  const long long C = N < JD_CHUNK ? (N + 31) / 32 * 32 : JD_CHUNK;
  double *yb = nullptr, *scr = nullptr, *Jrec = nullptr;
  int* status = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&yb, sizeof(double) * n * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&scr, sizeof(double) * Mech::NSC3 * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&Jrec, sizeof(double) * n * n * C, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&status, sizeof(int) * C, st);
  for (long long c0 = 0; e == cudaSuccess && c0 < N; c0 += C) {
    const long long m = N - c0 < C ? N - c0 : C;
    const unsigned g = (unsigned)((m + 127) / 128);
    jd_pack<Mech><<<g, 128, 0, st>>>(m, N, c0, y, yb);
    jd_part<Mech><<<g * Mech::NPART, 128, 0, st>>>(m, yb, aux + c0, scr, status);
    jd_sum<Mech><<<g, 128, 0, st>>>(m, yb, aux + c0, scr, status);
    jd_col<Mech><<<g * n, 128, 0, st>>>(m, scr, status, Jrec);
    jd_unpack<Mech><<<g, 128, 0, st>>>(m, N, c0, Jrec, status, J, flag);
    e = cudaGetLastError();
  }
  cudaFreeAsync(yb, st);
  cudaFreeAsync(scr, st);
  cudaFreeAsync(Jrec, st);
  cudaFreeAsync(status, st);
  return e;
}

using KH2 = SplitK<Tpc_h2_lidryer, ModelMech<mech_h2_lidryer::Traits>>;
using KDRM = SplitK<Tpc_drm19_class, ModelMech<mech_drm19_class::Traits>>;
using KGRI = SplitK<Tpc_gri53_class, LanesOf<Tpc_gri53_class>::GM>;   // n = 54 (split_big.cuh setup kernels)

}  // namespace

cudaError_t split_lu_diag(int n, long long N, double* M, int* piv, double* b, int* info, double* rec,
                          cudaStream_t st) {
  const unsigned g = (unsigned)((N * OCT + 127) / 128);
  switch (n) {
#define BDFB_LU_DIAG(NN) \
  case NN: split_lu_diag_kernel<NN><<<g, 128, 0, st>>>(N, M, piv, b, info, rec); break;
    BDFB_LU_DIAG(2) BDFB_LU_DIAG(4) BDFB_LU_DIAG(6) BDFB_LU_DIAG(8) BDFB_LU_DIAG(10) BDFB_LU_DIAG(12)
    BDFB_LU_DIAG(16) BDFB_LU_DIAG(22) BDFB_LU_DIAG(32)
#undef BDFB_LU_DIAG
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// scratch doubles per cell of the diagnostic's record pool (the caller rounds N up to a multiple of 32)
size_t split_lu_rec_doubles(int n) {
  return LU_STRIDE == 1 ? (size_t)((n * n + n + (n + 1) / 2 + 3) / 4 * 4) : (size_t)(n * n + 2 * n);
}

cudaError_t split_jac_diag(int mech, long long N, const double* y, const double* aux, double* J, int* flag,
                           cudaStream_t st) {
  switch (mech) {
    case BDFB_MODEL_MECH_H2: return jac_diag<Tpc_h2_lidryer>(N, y, aux, J, flag, st);
    case BDFB_MODEL_MECH_DRM19: return jac_diag<Tpc_drm19_class>(N, y, aux, J, flag, st);
    case BDFB_MODEL_MECH_GRI53: return jac_diag<Tpc_gri53_class>(N, y, aux, J, flag, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t split_geometry(int mech, int ls, int device, SplitGeom* gm) {
  if (ls != LS_DENSE) return split_mf_geometry(mech, ls, device, gm);
  switch (mech) {
    case BDFB_MODEL_MECH_H2: return KH2::geometry(device, gm);
    case BDFB_MODEL_MECH_DRM19: return KDRM::geometry(device, gm);
    case BDFB_MODEL_MECH_GRI53: return KGRI::geometry(device, gm);
  }
  return cudaErrorInvalidValue;
}

cudaError_t split_integrate(int mech, int ls, const Opts& o, double* y, const double* fext, const double* aux,
                            const double* atol, const SplitBufs& sb, const SplitGeom& gm, unsigned long long* counter,
                            Agg* agg, const CellStatsPtrs& cs, unsigned long long* h_live, int batch,
                            cudaStream_t st, int* launches, cudaEvent_t* events, double* phase_ms, cudaStream_t st2,
                            cudaEvent_t* xev) {
  if (ls != LS_DENSE)
    return split_mf_integrate(mech, ls, o, y, fext, aux, atol, sb, gm, counter, agg, cs, h_live, batch, st, launches,
                              events, phase_ms);
  switch (mech) {
    case BDFB_MODEL_MECH_H2:
      return KH2::run(o, y, fext, aux, atol, sb, gm, counter, agg, cs, h_live, batch, st, launches, events,
                       phase_ms, st2, xev);
    case BDFB_MODEL_MECH_DRM19:
      return KDRM::run(o, y, fext, aux, atol, sb, gm, counter, agg, cs, h_live, batch, st, launches, events,
                        phase_ms, st2, xev);
    case BDFB_MODEL_MECH_GRI53:
      return KGRI::run(o, y, fext, aux, atol, sb, gm, counter, agg, cs, h_live, batch, st, launches, events,
                        phase_ms, st2, xev);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bdfb
