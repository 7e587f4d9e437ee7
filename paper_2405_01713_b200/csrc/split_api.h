// split_api.h -- internal (not ABI) host interface of the SPLIT per-cell
// integrator (split.cu, bdf_split.cuh), used by bdfb.cu.  `mech` is a
// BDFB_MODEL_MECH_* id; functions return a CUDA error code
// (cudaErrorInvalidValue for an unknown id).
#pragma once
#include <cuda_runtime.h>

#include "bdf_cell.cuh"   // Opts, Agg, CellStatsPtrs

namespace bdfb {

struct SplitBufs;

struct SplitGeom {
  int rhs_grid;                            // resident blocks of K_rhs on the device
  int setup_grid;                          // blocks of the (grid-stride) Jacobian / LU kernels
  int vec_doubles, ts_doubles, jrec, lurec;   // doubles per slot of the VEC, TS, J and LU records
  int jscr;                                    // doubles per slot of the two-pass Jacobian scratch (0: none)
};

// ls: LS_DENSE | LS_DIAG | LS_GMRES (bdf_split.cuh); the matrix-free solvers are built in split_mf.cu
cudaError_t split_geometry(int mech, int ls, int device, SplitGeom* gm);
cudaError_t split_mf_geometry(int mech, int ls, int device, SplitGeom* gm);

// Integrate all o.ncells cells through the slot pool sb (host loop over
// K_ctl/K_rhs launch batches of `batch` iterations on st, one live-count read
// back per batch; synchronous).  launches: kernels enqueued.
// events: (SPLIT_PHASES + 2) * batch timing events (or NULL); phase_ms: device
// time of each phase (K_ctl, K_jac, K_lu, K_rhs) summed over the integrate.
// st2 (or NULL): a second stream on which K_jac and K_lu run, overlapping K_rhs
// (they touch disjoint slots); xev: 2 * batch ordering events for it.
constexpr int SPLIT_PHASES = 4;
cudaError_t split_integrate(int mech, int ls, const Opts& o, double* y, const double* fext, const double* aux,
                            const double* atol, const SplitBufs& sb, const SplitGeom& gm, unsigned long long* counter,
                            Agg* agg, const CellStatsPtrs& cs, unsigned long long* h_live, int batch,
                            cudaStream_t st, int* launches, cudaEvent_t* events, double* phase_ms,
                            cudaStream_t st2, cudaEvent_t* xev);

cudaError_t split_mf_integrate(int mech, int ls, const Opts& o, double* y, const double* fext, const double* aux,
                               const double* atol, const SplitBufs& sb, const SplitGeom& gm,
                               unsigned long long* counter, Agg* agg, const CellStatsPtrs& cs,
                               unsigned long long* h_live, int batch, cudaStream_t st, int* launches,
                               cudaEvent_t* events, double* phase_ms);

// K_rhs launch and occupancy (rhs.cu, the -fmad=true translation unit; explicit instantiations for both
// mechanisms and the three linear solvers)
template <class Mech, class GM, int LS>
cudaError_t split_rhs_run(unsigned grid, cudaStream_t st, const SplitBufs& b, int it);
template <class Mech, class GM, int LS>
cudaError_t split_rhs_occupancy(int* blocks_per_sm);
// f = R(y) + F with the K_rhs code (rhs.cu), YC layout
cudaError_t tpc_eval_rhs(int mech, long long N, const double* y, const double* fext, const double* aux, double* f,
                         int* status, cudaStream_t st);

// LU diagnostic with the SPLIT path's routines (oct_factor + the Newton
// solve's substitutions); n in {2,4,6,8,10,12,16,22,32}; rec: N *
// split_lu_rec_doubles(n) doubles of device scratch.
cudaError_t split_lu_diag(int n, long long N, double* M, int* piv, double* b, int* info, double* rec,
                          cudaStream_t st);
size_t split_lu_rec_doubles(int n);
// The SPLIT path's two-pass generated Jacobian (jac_part / jac_sum / jac_col) on N cells in chunks of 65536:
// y[k N + c] in, J[(i n + j) N + c] out (cells whose T <= 0 are left untouched and set *flag, if given, to 1);
// device scratch allocated and freed on st.  The Jacobian diagnostic, and the global-norm mode's J for n = 54.
cudaError_t split_jac_diag(int mech, long long N, const double* y, const double* aux, double* J, int* flag,
                           cudaStream_t st);

}  // namespace bdfb
