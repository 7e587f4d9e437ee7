// split_mf.cu -- the SPLIT per-cell integrator with the matrix-free linear solvers of the Newton
// iteration and the SPLIT-organised explicit ERK (LS_ERK, erk_split.cuh); originally: the matrix-free solvers of the Newton
// iteration: CVDiag (LS_DIAG) and inexact Newton-Krylov GMRES with the difference-quotient Jv
// (LS_GMRES, approaches 1A/1B).  Same slot pool and kernels as split.cu minus the setup
// kernels (K_jac, K_lu); a separate translation unit of libbdfb.so so that the dense build is unchanged.
#include "../../include/bdfb.h"
#include "gen/mech_drm19_class.cuh"
#include "gen/mech_h2_lidryer.cuh"
#include "gen/tpc_drm19_class.cuh"
#include "gen/tpc_h2_lidryer.cuh"
#include "mech_model.cuh"
#include "split_run.cuh"

namespace bdfb {
namespace {
template <int LS>
using KH2L = SplitK<Tpc_h2_lidryer, ModelMech<mech_h2_lidryer::Traits>, LS>;
template <int LS>
using KDRML = SplitK<Tpc_drm19_class, ModelMech<mech_drm19_class::Traits>, LS>;
template <int LS>
using KGRIL = SplitK<Tpc_gri53_class, LanesOf<Tpc_gri53_class>::GM, LS>;
}  // namespace

cudaError_t split_mf_geometry(int mech, int ls, int device, SplitGeom* gm) {
  switch (mech * 4 + ls) {
    case BDFB_MODEL_MECH_H2 * 4 + LS_DIAG: return KH2L<LS_DIAG>::geometry(device, gm);
    case BDFB_MODEL_MECH_H2 * 4 + LS_GMRES: return KH2L<LS_GMRES>::geometry(device, gm);
    case BDFB_MODEL_MECH_DRM19 * 4 + LS_DIAG: return KDRML<LS_DIAG>::geometry(device, gm);
    case BDFB_MODEL_MECH_DRM19 * 4 + LS_GMRES: return KDRML<LS_GMRES>::geometry(device, gm);
    case BDFB_MODEL_MECH_GRI53 * 4 + LS_DIAG: return KGRIL<LS_DIAG>::geometry(device, gm);
    case BDFB_MODEL_MECH_GRI53 * 4 + LS_GMRES: return KGRIL<LS_GMRES>::geometry(device, gm);
    case BDFB_MODEL_MECH_H2 * 4 + LS_ERK: return KH2L<LS_ERK>::geometry(device, gm);
    case BDFB_MODEL_MECH_DRM19 * 4 + LS_ERK: return KDRML<LS_ERK>::geometry(device, gm);
    case BDFB_MODEL_MECH_GRI53 * 4 + LS_ERK: return KGRIL<LS_ERK>::geometry(device, gm);
  }
  return cudaErrorInvalidValue;
}

cudaError_t split_mf_integrate(int mech, int ls, const Opts& o, double* y, const double* fext, const double* aux,
                               const double* atol, const SplitBufs& sb, const SplitGeom& gm,
                               unsigned long long* counter, Agg* agg, const CellStatsPtrs& cs,
                               unsigned long long* h_live, int batch, cudaStream_t st, int* launches,
                               cudaEvent_t* events, double* phase_ms) {
#define BDFB_MF_RUN(K) \
  K::run(o, y, fext, aux, atol, sb, gm, counter, agg, cs, h_live, batch, st, launches, events, phase_ms, nullptr, nullptr)
  switch (mech * 4 + ls) {
    case BDFB_MODEL_MECH_H2 * 4 + LS_DIAG: return BDFB_MF_RUN(KH2L<LS_DIAG>);
    case BDFB_MODEL_MECH_H2 * 4 + LS_GMRES: return BDFB_MF_RUN(KH2L<LS_GMRES>);
    case BDFB_MODEL_MECH_DRM19 * 4 + LS_DIAG: return BDFB_MF_RUN(KDRML<LS_DIAG>);
    case BDFB_MODEL_MECH_DRM19 * 4 + LS_GMRES: return BDFB_MF_RUN(KDRML<LS_GMRES>);
    case BDFB_MODEL_MECH_GRI53 * 4 + LS_DIAG: return BDFB_MF_RUN(KGRIL<LS_DIAG>);
    case BDFB_MODEL_MECH_GRI53 * 4 + LS_GMRES: return BDFB_MF_RUN(KGRIL<LS_GMRES>);
    case BDFB_MODEL_MECH_H2 * 4 + LS_ERK: return BDFB_MF_RUN(KH2L<LS_ERK>);
    case BDFB_MODEL_MECH_DRM19 * 4 + LS_ERK: return BDFB_MF_RUN(KDRML<LS_ERK>);
    case BDFB_MODEL_MECH_GRI53 * 4 + LS_ERK: return BDFB_MF_RUN(KGRIL<LS_ERK>);
  }
#undef BDFB_MF_RUN
  return cudaErrorInvalidValue;
}

}  // namespace bdfb
