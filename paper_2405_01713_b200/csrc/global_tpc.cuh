// global_tpc.cuh -- thread-per-cell device kernels of the global-norm mode
// (row a12) for the mechanism models: the lockstep batch advances every cell
// in every kernel, so one thread per cell with the state in cell-minor SoA
// (element e of cell c at [e * N + c]) streams HBM fully coalesced.
//   gt_rhs:   f = R(y) + F, the generated straight-line RHS (gen/tpc_<mech>.cuh)
//   gt_setup: [J = dR/dy (generated analytic Jacobian)]; M = I - gamma J and
//             LU with partial pivoting (tpc_factor, left-looking, bit-identical
//             to the listing's LU_FACTOR, reading R16); factors in pivoted row
//             positions, perm[i] (original row at position i), 1/U_ii
//   gt_solve: b = M^{-1}(-del) (tpc_solve = LU_SOLVE), the stale-gamma scale,
//             acor += b, tmp = b
// Same operations as the group kernels of global_mode.cuh (glu_factor /
// glu_solve implement the same LU_FACTOR / LU_SOLVE), so the lockstep
// decisions and the end states are unchanged up to the RHS rounding.
#pragma once
#include "bdf_tpc.cuh"

namespace bdfb {

template <class Mech>
__global__ void __launch_bounds__(128) gt_rhs(long long N, const double* y, const double* fext, const double* aux,
                                              double* f, int* flag) {
  constexpr int NN = Mech::N;
  const long long c = (long long)blockIdx.x * 128 + threadIdx.x;
  int rv = 0;
  if (c < N) {
    double yv[NN], fv[NN];
#pragma unroll
    for (int k = 0; k < NN; ++k) yv[k] = y[(long long)k * N + c];
    rv = Mech::rhs(yv, aux ? aux[c] : 0.0, fv);
#pragma unroll
    for (int k = 0; k < NN; ++k) f[(long long)k * N + c] = fv[k] + (fext ? fext[(long long)k * N + c] : 0.0);
  }
  if (__any_sync(0xffffffffu, rv != 0) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <class Mech>
__global__ void __launch_bounds__(128) gt_setup(long long N, int jbad, double gamma, const double* y,
                                                const double* aux, double* J, double* LU, int* perm, double* invd,
                                                int* flag) {
  constexpr int NN = Mech::N;
  const long long c = (long long)blockIdx.x * 128 + threadIdx.x;
  int bad = 0;
  if (c < N) {
    if (jbad) bad = Mech::template jac<0>(y + c, aux ? aux[c] : 0.0, J + c, LU + c, N);   // LU area = scratch
    if (!bad) bad = tpc_factor<NN, true, 0>(J + c, LU + c, invd + c, perm + c, N, gamma, nullptr);
  }
  if (__any_sync(0xffffffffu, bad != 0) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <class Mech>
__global__ void __launch_bounds__(128) gt_solve(long long N, double sc2, const double* LU, const int* perm,
                                                const double* invd, const double* del, double* acor, double* tmp) {
  constexpr int NN = Mech::N;
  const long long c = (long long)blockIdx.x * 128 + threadIdx.x;
  if (c >= N) return;
  double x[NN];
  tpc_solve<NN, true, 0>(LU + c, invd + c, perm + c, del + c, N, x);
#pragma unroll
  for (int k = 0; k < NN; ++k) {
    const double b = (sc2 != 1.0) ? sc2 * x[k] : x[k];
    const long long e = (long long)k * N + c;
    acor[e] = acor[e] + b;
    tmp[e] = b;
  }
}

}  // namespace bdfb
