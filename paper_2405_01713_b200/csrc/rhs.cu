// rhs.cu -- the generated thread-per-cell reaction RHS kernels of the SPLIT path (K_rhs, bdf_split.cuh) and
// the RHS diagnostic that runs the same code; a translation unit of libbdfb.so of its own, so that its
// compile flags can differ from the integrator's.  Contraction (-fmad=true: a*b + c as one DFMA in the
// generated sums of products, within the R19 parity bar) was measured 3% SLOWER for K_rhs on C4 (ncu:
// more spills at 168 registers; profiles/r2/history.md), so the unit builds with -fmad=false like the rest.
#include <cuda_runtime.h>
#include <stdlib.h>

#include "../../include/bdfb.h"
#include "bdf_split.cuh"
#include "gen/mech_drm19_class.cuh"
#include "gen/mech_h2_lidryer.cuh"
#include "gen/tpc_drm19_class.cuh"
#include "gen/tpc_h2_lidryer.cuh"
#include "gen/tpc_gri53_class.cuh"
#include "mech_model.cuh"
#include "split_api.h"
#include "split_big.cuh"

namespace bdfb {

// K_rhs organisation (RhsVar in bdf_split.cuh): 3 (e^{-g/RT} in shared memory: C4 K_rhs 1013 -> 930 ms, no
// spills) when its 2K doubles per thread fit 64 KB per block, else 0 (free-running 128-thread blocks);
// BDFB_SPLIT_RHS_VAR = 0 forces 0.  VARs 1, 2 and 4 (block-synchronous trips, 16 warps/SM) measured equal or
// slower in round 2 (profiles/r2/history.md) and are no longer instantiated (they tripled the unit's compile time).
template <class Mech>
__host__ __device__ constexpr bool rhs_sm_fits() {
  return 2 * Mech::K * RhsVar<3>::BLOCK * 8 <= 64 * 1024;
}
template <class Mech>
static int rhs_var() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BDFB_SPLIT_RHS_VAR");
    v = (rhs_sm_fits<Mech>() && !(e && atoi(e) == 0)) ? 3 : 0;
  }
  return v;
}

template <class Mech>
constexpr size_t rhs_sm_bytes() {
  return sizeof(double) * 2 * Mech::K * RhsVar<3>::BLOCK;
}

template <class Mech, class GM, int LS>
cudaError_t split_rhs_run(unsigned grid, cudaStream_t st, const SplitBufs& b, int it) {
  if constexpr (rhs_sm_fits<Mech>()) {
    if (rhs_var<Mech>() == 3) {
      split_rhs_kernel<Mech, GM, LS, 3><<<grid, RhsVar<3>::BLOCK, rhs_sm_bytes<Mech>(), st>>>(b, it);
      return cudaSuccess;
    }
  }
  split_rhs_kernel<Mech, GM, LS, 0><<<grid, RhsVar<0>::BLOCK, 0, st>>>(b, it);
  return cudaSuccess;
}

// resident blocks per SM of the selected organisation, expressed in 128-thread (BDFB_SPLIT_BLOCK) units so
// that the caller's grid (nsm x blocks) covers the same threads
template <class Mech, class GM, int LS>
cudaError_t split_rhs_occupancy(int* blocks_per_sm) {
  if constexpr (rhs_sm_fits<Mech>()) {
    if (rhs_var<Mech>() == 3) {
      cudaError_t e = cudaFuncSetAttribute(split_rhs_kernel<Mech, GM, LS, 3>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rhs_sm_bytes<Mech>());
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, split_rhs_kernel<Mech, GM, LS, 3>,
                                                          RhsVar<3>::BLOCK, rhs_sm_bytes<Mech>());
      return e;
    }
  }
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, split_rhs_kernel<Mech, GM, LS, 0>,
                                                       RhsVar<0>::BLOCK, 0);
}

#define BDFB_RHS_INST(M, G, LS)                                                                       \
  template cudaError_t split_rhs_run<M, G, LS>(unsigned, cudaStream_t, const SplitBufs&, int);       \
  template cudaError_t split_rhs_occupancy<M, G, LS>(int*);
using GH2 = ModelMech<mech_h2_lidryer::Traits>;
using GDRM = ModelMech<mech_drm19_class::Traits>;
BDFB_RHS_INST(Tpc_h2_lidryer, GH2, LS_DENSE)
BDFB_RHS_INST(Tpc_h2_lidryer, GH2, LS_DIAG)
BDFB_RHS_INST(Tpc_h2_lidryer, GH2, LS_GMRES)
BDFB_RHS_INST(Tpc_drm19_class, GDRM, LS_DENSE)
BDFB_RHS_INST(Tpc_drm19_class, GDRM, LS_DIAG)
BDFB_RHS_INST(Tpc_drm19_class, GDRM, LS_GMRES)
using GGRI = LanesOf<Tpc_gri53_class>::GM;
BDFB_RHS_INST(Tpc_gri53_class, GGRI, LS_DENSE)
BDFB_RHS_INST(Tpc_gri53_class, GGRI, LS_DIAG)
BDFB_RHS_INST(Tpc_gri53_class, GGRI, LS_GMRES)
BDFB_RHS_INST(Tpc_h2_lidryer, GH2, 3)      // LS_ERK
BDFB_RHS_INST(Tpc_drm19_class, GDRM, 3)
BDFB_RHS_INST(Tpc_gri53_class, GGRI, 3)
#undef BDFB_RHS_INST

// f = R(y) + F for N cells (YC), the K_rhs code path (diagnostic entry point bdfb_eval_rhs)
template <class Mech>
__global__ void __launch_bounds__(128) eval_rhs_kernel(long long N, const double* y, const double* fext,
                                                       const double* aux, double* f, int* status, int use_sm) {
  constexpr int n = Mech::N;
  const long long c = blockIdx.x * 128ll + threadIdx.x;
  if (c >= N) return;
  double yv[n], fv[n];
#pragma unroll
  for (int i = 0; i < n; ++i) yv[i] = y[(long long)i * N + c];
  int rv;
  if constexpr (rhs_sm_fits<Mech>()) {
    if (use_sm) {   // the device function K_rhs runs (the host's RhsVar choice)
      extern __shared__ double rsm[];
      rv = Mech::template rhs_sm<128>(yv, aux[c], fv, rsm + threadIdx.x);
    } else {
      rv = Mech::rhs(yv, aux[c], fv);
    }
  } else {
    rv = Mech::rhs(yv, aux[c], fv);
  }
#pragma unroll
  for (int i = 0; i < n; ++i) f[(long long)i * N + c] = fv[i] + (fext ? fext[(long long)i * N + c] : 0.0);
  if (status) status[c] = rv;
}

template <class Mech>
static void launch_eval_rhs(unsigned g, long long N, const double* y, const double* fext, const double* aux, double* f,
                            int* status, cudaStream_t st) {
  const int sm = rhs_var<Mech>() >= 3;
  const size_t bytes = sm ? sizeof(double) * 2 * Mech::K * 128 : 0;
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(eval_rhs_kernel<Mech>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  eval_rhs_kernel<Mech><<<g, 128, bytes, st>>>(N, y, fext, aux, f, status, sm);
}

cudaError_t tpc_eval_rhs(int mech, long long N, const double* y, const double* fext, const double* aux, double* f,
                         int* status, cudaStream_t st) {
  const unsigned g = (unsigned)((N + 127) / 128);
  switch (mech) {
    case BDFB_MODEL_MECH_H2: launch_eval_rhs<Tpc_h2_lidryer>(g, N, y, fext, aux, f, status, st); break;
    case BDFB_MODEL_MECH_DRM19:
      launch_eval_rhs<Tpc_drm19_class>(g, N, y, fext, aux, f, status, st);
      break;
    case BDFB_MODEL_MECH_GRI53:
      launch_eval_rhs<Tpc_gri53_class>(g, N, y, fext, aux, f, status, st);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace bdfb
