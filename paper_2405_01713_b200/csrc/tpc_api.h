// tpc_api.h -- internal (not ABI) host interface of the thread-per-cell
// mechanism kernels in tpc.cu, used by bdfb.cu.  `mech` is a BDFB_MODEL_MECH_*
// id; all functions return a CUDA error code (cudaErrorInvalidValue for an
// unknown id) and enqueue on `st`.
#pragma once
#include <cuda_runtime.h>
#include "bdf_cell.cuh"   // Opts, Agg, CellStatsPtrs

namespace bdfb {
// resident slots of the persistent grid on `device` (min of occupancy and
// ncells), workspace doubles and ints per slot
cudaError_t tpc_geometry(int mech, int device, long long ncells, long long* slots, long long* doubles_per_slot,
                         long long* ints_per_slot);
cudaError_t tpc_integrate(int mech, const Opts& o, double* y, const double* fext, const double* aux,
                          const double* atol, double* ws, int* iws, long long slots, unsigned long long* counter,
                          Agg* agg, const CellStatsPtrs& cs, cudaStream_t st);
// f = R(y) + F (J == nullptr) or J = dR/dy for N cells, YC layout
cudaError_t tpc_eval(int mech, long long N, const double* y, const double* fext, const double* aux, double* f,
                     int* status, double* J, cudaStream_t st);
// batched LU factor + solve (n >= 5; diagnostic entry point, the integrator's routine)
cudaError_t tpc_lu(int n, long long N, double* M, int* piv, double* b, int* info, cudaStream_t st);
}  // namespace bdfb
