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
