// tpc.cu -- thread-per-cell mechanism kernels (bdf_tpc.cuh) and their host
// launchers (tpc_api.h); a translation unit of libbdfb.so.
#include <cuda_runtime.h>

#include "../../include/bdfb.h"
#include "bdf_tpc.cuh"
#include "gen/mech_drm19_class.cuh"
#include "gen/mech_h2_lidryer.cuh"
#include "gen/tpc_drm19_class.cuh"
#include "gen/tpc_h2_lidryer.cuh"
#include "mech_model.cuh"
#include "tpc_api.h"
#include "split_api.h"

namespace bdfb {

template <class Mech>
__global__ void __launch_bounds__(128) eval_tpc_kernel(long long N, const double* y, const double* fext,
                                                       const double* aux, double* f, int* status, double* J,
                                                       double* sc) {
  constexpr int n = Mech::N;
  const long long c = blockIdx.x * 128ll + threadIdx.x;
  if (c >= N) return;
  if (J == nullptr) {
    double yv[n], fv[n];
#pragma unroll
    for (int i = 0; i < n; ++i) {
      yv[i] = y[(long long)i * N + c];
      fv[i] = 0.0;
    }
    const int rv = Mech::rhs(yv, aux[c], fv);
#pragma unroll
    for (int i = 0; i < n; ++i) f[(long long)i * N + c] = fv[i] + (fext ? fext[(long long)i * N + c] : 0.0);
    if (status) status[c] = rv;
  } else {
    Mech::template jac<0>(y + c, aux[c], J + c, sc + c, N);
  }
}

template <int NN>
__global__ void __launch_bounds__(128) lu_tpc_kernel(long long N, double* M, int* piv, double* b, int* info,
                                                     int* perm, double* invd) {
  const long long c = blockIdx.x * 128ll + threadIdx.x;
  if (c >= N) return;
  const int inf = tpc_factor<NN, false, 0>(M + c, M + c, invd + c, perm + c, N, 0.0, piv + c);
  info[c] = inf;
  if (!inf) {
    double x[NN];
    tpc_solve<NN, false, 0>(M + c, invd + c, perm + c, b + c, N, x);
#pragma unroll
    for (int i = 0; i < NN; ++i) b[(long long)i * N + c] = x[i];
  }
}

namespace {
// thread-per-cell model and the group model of its warp-cooperative stages
template <class Mech>
struct GroupOf;
template <>
struct GroupOf<Tpc_h2_lidryer> {
  using type = ModelMech<mech_h2_lidryer::Traits>;
};
template <>
struct GroupOf<Tpc_drm19_class> {
  using type = ModelMech<mech_drm19_class::Traits>;
};
template <class Mech>
constexpr size_t smem_of() { return tpc_smem_bytes<Mech, typename GroupOf<Mech>::type>(); }
template <class Mech>
constexpr auto kernel_of() { return integrate_tpc_kernel<Mech, typename GroupOf<Mech>::type>; }

template <class Mech>
cudaError_t geometry(int device, long long ncells, long long* slots, long long* dps, long long* ips) {
  auto kern = kernel_of<Mech>();
  const size_t kSmem = smem_of<Mech>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
  if (e != cudaSuccess) return e;
  int nsm = 0, per_sm = 0;
  if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BDFB_TPC_BLOCK, kSmem)) != cudaSuccess)
    return e;
  long long grid = (long long)nsm * per_sm;
  const long long need = (ncells + BDFB_TPC_BLOCK - 1) / BDFB_TPC_BLOCK;
  if (grid > need) grid = need;
  *slots = grid * BDFB_TPC_BLOCK;
  *dps = TWs<Mech::N>::DOUBLES;
  *ips = TWs<Mech::N>::INTS;
  return cudaSuccess;
}

template <class Mech>
cudaError_t integrate(const Opts& o, double* y, const double* fext, const double* aux, const double* atol,
                      double* ws, int* iws, long long slots, unsigned long long* counter, Agg* agg,
                      const CellStatsPtrs& cs, cudaStream_t st) {
  const unsigned grid = (unsigned)(slots / BDFB_TPC_BLOCK);
  kernel_of<Mech>()<<<grid, BDFB_TPC_BLOCK, smem_of<Mech>(), st>>>(o, y, fext, aux, atol, ws, iws, counter, agg, cs);
  return cudaGetLastError();
}

template <class Mech>
cudaError_t eval(long long N, const double* y, const double* fext, const double* aux, double* f, int* status,
                 double* J, cudaStream_t st) {
  double* sc = nullptr;
  cudaError_t e;
  if (J && (e = cudaMallocAsync(&sc, sizeof(double) * Mech::NSC * (size_t)N, st)) != cudaSuccess) return e;
  eval_tpc_kernel<Mech><<<(unsigned)((N + 127) / 128), 128, 0, st>>>(N, y, fext, aux, f, status, J, sc);
  e = cudaGetLastError();
  if (sc) cudaFreeAsync(sc, st);
  return e;
}

template <int NN>
cudaError_t lu(long long N, double* M, int* piv, double* b, int* info, cudaStream_t st) {
  int* perm = nullptr;
  double* invd = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync(&perm, sizeof(int) * NN * (size_t)N, st)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&invd, sizeof(double) * NN * (size_t)N, st)) != cudaSuccess) return e;
  lu_tpc_kernel<NN><<<(unsigned)((N + 127) / 128), 128, 0, st>>>(N, M, piv, b, info, perm, invd);
  e = cudaGetLastError();
  cudaFreeAsync(perm, st);
  cudaFreeAsync(invd, st);
  return e;
}
}  // namespace

cudaError_t tpc_geometry(int mech, int device, long long ncells, long long* slots, long long* dps, long long* ips) {
  switch (mech) {
    case BDFB_MODEL_MECH_H2: return geometry<Tpc_h2_lidryer>(device, ncells, slots, dps, ips);
    case BDFB_MODEL_MECH_DRM19: return geometry<Tpc_drm19_class>(device, ncells, slots, dps, ips);
  }
  return cudaErrorInvalidValue;
}

cudaError_t tpc_integrate(int mech, const Opts& o, double* y, const double* fext, const double* aux,
                          const double* atol, double* ws, int* iws, long long slots, unsigned long long* counter,
                          Agg* agg, const CellStatsPtrs& cs, cudaStream_t st) {
  switch (mech) {
    case BDFB_MODEL_MECH_H2:
      return integrate<Tpc_h2_lidryer>(o, y, fext, aux, atol, ws, iws, slots, counter, agg, cs, st);
    case BDFB_MODEL_MECH_DRM19:
      return integrate<Tpc_drm19_class>(o, y, fext, aux, atol, ws, iws, slots, counter, agg, cs, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t tpc_eval(int mech, long long N, const double* y, const double* fext, const double* aux, double* f,
                     int* status, double* J, cudaStream_t st) {
  if (J == nullptr) return tpc_eval_rhs(mech, N, y, fext, aux, f, status, st);   // the K_rhs code (rhs.cu)
  switch (mech) {
    case BDFB_MODEL_MECH_H2: return eval<Tpc_h2_lidryer>(N, y, fext, aux, f, status, J, st);
    case BDFB_MODEL_MECH_DRM19: return eval<Tpc_drm19_class>(N, y, fext, aux, f, status, J, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t tpc_lu(int n, long long N, double* M, int* piv, double* b, int* info, cudaStream_t st) {
  switch (n) {
    case 5: return lu<5>(N, M, piv, b, info, st);
    case 6: return lu<6>(N, M, piv, b, info, st);
    case 7: return lu<7>(N, M, piv, b, info, st);
    case 8: return lu<8>(N, M, piv, b, info, st);
    case 10: return lu<10>(N, M, piv, b, info, st);
    case 12: return lu<12>(N, M, piv, b, info, st);
    case 16: return lu<16>(N, M, piv, b, info, st);
    case 22: return lu<22>(N, M, piv, b, info, st);
    case 32: return lu<32>(N, M, piv, b, info, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bdfb
