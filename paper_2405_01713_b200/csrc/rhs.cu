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

// K_rhs organisation (RhsVar in bdf_split.cuh): BDFB_SPLIT_RHS_VAR = 0 | 1 | 2 (default 0)
static int rhs_var() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BDFB_SPLIT_RHS_VAR");
    v = e ? atoi(e) : 0;
    if (v < 0 || v > 2) v = 0;
  }
  return v;
}

template <class Mech, class GM, int LS>
cudaError_t split_rhs_run(unsigned grid, cudaStream_t st, const SplitBufs& b, int it) {
  switch (rhs_var()) {
    case 1: split_rhs_kernel<Mech, GM, LS, 1><<<grid, RhsVar<1>::BLOCK, 0, st>>>(b, it); break;
    case 2: split_rhs_kernel<Mech, GM, LS, 2><<<grid, RhsVar<2>::BLOCK, 0, st>>>(b, it); break;
    default: split_rhs_kernel<Mech, GM, LS, 0><<<grid, RhsVar<0>::BLOCK, 0, st>>>(b, it);
  }
  return cudaSuccess;
}

// resident blocks per SM of the selected organisation, expressed in 128-thread (BDFB_SPLIT_BLOCK) units so
// that the caller's grid (nsm x blocks) covers the same threads
template <class Mech, class GM, int LS>
cudaError_t split_rhs_occupancy(int* blocks_per_sm) {
  cudaError_t e;
  switch (rhs_var()) {
    case 1: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, split_rhs_kernel<Mech, GM, LS, 1>,
                                                            RhsVar<1>::BLOCK, 0); break;
    case 2: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, split_rhs_kernel<Mech, GM, LS, 2>,
                                                            RhsVar<2>::BLOCK, 0); break;
    default: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, split_rhs_kernel<Mech, GM, LS, 0>,
                                                             RhsVar<0>::BLOCK, 0);
  }
  return e;
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
#undef BDFB_RHS_INST

// f = R(y) + F for N cells (YC), the K_rhs code path (diagnostic entry point bdfb_eval_rhs)
template <class Mech>
__global__ void __launch_bounds__(128) eval_rhs_kernel(long long N, const double* y, const double* fext,
                                                       const double* aux, double* f, int* status) {
  constexpr int n = Mech::N;
  const long long c = blockIdx.x * 128ll + threadIdx.x;
  if (c >= N) return;
  double yv[n], fv[n];
#pragma unroll
  for (int i = 0; i < n; ++i) yv[i] = y[(long long)i * N + c];
  const int rv = Mech::rhs(yv, aux[c], fv);
#pragma unroll
  for (int i = 0; i < n; ++i) f[(long long)i * N + c] = fv[i] + (fext ? fext[(long long)i * N + c] : 0.0);
  if (status) status[c] = rv;
}

cudaError_t tpc_eval_rhs(int mech, long long N, const double* y, const double* fext, const double* aux, double* f,
                         int* status, cudaStream_t st) {
  const unsigned g = (unsigned)((N + 127) / 128);
  switch (mech) {
    case BDFB_MODEL_MECH_H2: eval_rhs_kernel<Tpc_h2_lidryer><<<g, 128, 0, st>>>(N, y, fext, aux, f, status); break;
    case BDFB_MODEL_MECH_DRM19:
      eval_rhs_kernel<Tpc_drm19_class><<<g, 128, 0, st>>>(N, y, fext, aux, f, status);
      break;
    case BDFB_MODEL_MECH_GRI53:
      eval_rhs_kernel<Tpc_gri53_class><<<g, 128, 0, st>>>(N, y, fext, aux, f, status);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace bdfb
