// erk_api.h -- internal (not ABI) host interface of the explicit ERK integrator (erk.cu), used by
// bdfb.cu.  `mech` is a BDFB_MODEL_MECH_* id; functions return a CUDA error code
// (cudaErrorInvalidValue for an unknown id) and enqueue on `st`.
#pragma once
#include <cuda_runtime.h>
#include "bdf_cell.cuh"   // Opts, Agg, CellStatsPtrs

namespace bdfb {
// threads of the persistent grid (resident blocks on `device`, at most what ncells needs) and the
// workspace doubles per thread
cudaError_t erk_geometry(int mech, int device, long long ncells, long long* threads, long long* doubles_per_thread);
cudaError_t erk_integrate(int mech, const Opts& o, double* y, const double* fext, const double* aux,
                          const double* atol, double* ws, long long threads, unsigned long long* counter, Agg* agg,
                          const CellStatsPtrs& cs, cudaStream_t st);
}  // namespace bdfb
