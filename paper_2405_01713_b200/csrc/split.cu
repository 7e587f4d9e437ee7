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

namespace bdfb {
namespace {

template <class Mech, class GM>
struct SplitK {
  using SP = Split<Mech, GM>;
  static constexpr size_t ctl_smem() {
    return BDFB_SPLIT_TS_SMEM ? sizeof(double) * (size_t)TS_STRIDE * BDFB_SPLIT_CTL_BLOCK : 0;
  }
  static constexpr size_t jac_smem() {
    return sizeof(double) * (size_t)(GM::SG + GM::JG + GM::N * (GM::N | 1)) * (BDFB_SPLIT_BLOCK / GM::G);
  }

  static cudaError_t geometry(int device, SplitGeom* gm) {
    cudaError_t e;
    const int sm = (int)ctl_smem();
    if ((e = cudaFuncSetAttribute(split_ctl_kernel<Mech, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  sm > 110 * 1024 ? sm : 110 * 1024)) != cudaSuccess)
      return e;
    int nsm = 0, pr = 0;
    if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pr, split_rhs_kernel<Mech, GM>, BDFB_SPLIT_BLOCK, 0)) !=
        cudaSuccess)
      return e;
    if (pr < 1) return cudaErrorInvalidConfiguration;
    if (jac_smem() > 48 * 1024 &&
        (e = cudaFuncSetAttribute(split_jac_kernel<Mech, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)jac_smem())) != cudaSuccess)
      return e;
    gm->rhs_grid = nsm * pr;
    gm->setup_grid = nsm * 8;
    gm->vec_doubles = SP::D;
    gm->ts_doubles = TS_STRIDE;
    gm->jrec = SP::JREC;
    gm->lurec = SP::LUREC;
    return cudaSuccess;
  }

  static cudaError_t run(const Opts& o, double* y, const double* fext, const double* aux, const double* atol,
                         const SplitBufs& b, const SplitGeom& gm, unsigned long long* counter, Agg* agg,
                         const CellStatsPtrs& cs, unsigned long long* h_live, int batch, cudaStream_t st,
                         int* launches, cudaEvent_t* events, double* phase_ms, cudaStream_t st2,
                         cudaEvent_t* xev) {
    const long long S = b.slots;
    const unsigned blk = BDFB_SPLIT_BLOCK;
    const unsigned gs = (unsigned)((S + blk - 1) / blk);            // one thread per slot / list entry
    const unsigned gctl = (unsigned)((S + BDFB_SPLIT_CTL_BLOCK - 1) / BDFB_SPLIT_CTL_BLOCK);
    // setup kernels: persistent grids (grid-stride over the lists): K_jac one group of G lanes per entry,
    // K_lu one group of 8 lanes per entry
    unsigned gjac = (unsigned)((S * GM::G + blk - 1) / blk);
    if (gjac > (unsigned)gm.setup_grid) gjac = (unsigned)gm.setup_grid;
    const unsigned ginit = gs < (unsigned)gm.setup_grid ? gs : (unsigned)gm.setup_grid;   // grid-stride over the list
    unsigned gdq = (unsigned)gm.rhs_grid;   // K_dqjac: grid-stride over (entry, column)
    unsigned glu = (unsigned)((S * OCT + blk - 1) / blk);
    if (glu > (unsigned)gm.setup_grid) glu = (unsigned)gm.setup_grid;
    unsigned grhs = (unsigned)gm.rhs_grid;
    if (grhs > gs) grhs = gs;
    if (const char* g = getenv("BDFB_SPLIT_RHS_FULLGRID"))   // experiments: one thread per slot
      if (atoi(g) == 1) grhs = gs;
    size_t sm = ctl_smem();
    if (const char* pad = getenv("BDFB_SPLIT_CTL_SMEM")) {  // experiments: cap the resident K_ctl blocks
      const size_t want = (size_t)strtoul(pad, nullptr, 10);
      if (want > sm) sm = want;
    }
    split_init_kernel<Mech, GM><<<gs, blk, 0, st>>>(b);
    int n = 1;
    cudaError_t e;
    for (int i = 0; i < SPLIT_PHASES; ++i) phase_ms[i] = 0.0;
    const bool ovl = st2 != nullptr;   // K_jac + K_lu on st2, overlapping K_rhs (disjoint slots)
    if (ovl) grhs = grhs * 2 / 3 > 0 ? grhs * 2 / 3 : 1;   // leave registers for the setup kernels
    cudaEvent_t last_l = nullptr;
    for (int it = 0;;) {
      int k = 0;
      for (; k < batch; ++k, ++it) {
        cudaEvent_t* ev = events + k * (SPLIT_PHASES + 2);
        if (ovl && last_l) cudaStreamWaitEvent(st, last_l, 0);
        if (events) cudaEventRecord(ev[0], st);
        split_ctl_kernel<Mech, GM><<<gctl, BDFB_SPLIT_CTL_BLOCK, sm, st>>>(o, b, it, y, fext, aux, atol, counter, agg, cs);
#if BDFB_SPLIT_INIT_KERNEL
        split_init_cells_kernel<Mech, GM><<<ginit, blk, 0, st>>>(o, b, it, y, fext, aux, atol, counter, agg, cs);
        ++n;
#endif
        if (events) cudaEventRecord(ev[1], st);
        cudaStream_t ss = st;
        if (ovl) {
          cudaEventRecord(xev[2 * k], st);
          cudaStreamWaitEvent(st2, xev[2 * k], 0);
          ss = st2;
          if (events) cudaEventRecord(ev[5], st2);
        }
        if (b.jac_dq)
          split_dqjac_kernel<Mech, GM><<<gdq, blk, 0, ss>>>(b, it);
        else
          split_jac_kernel<Mech, GM><<<gjac, blk, jac_smem(), ss>>>(b, it);
        if (events) cudaEventRecord(ev[2], ss);
        split_lu_kernel<Mech, GM><<<glu, blk, 0, ss>>>(b, it);
        if (events) cudaEventRecord(ev[3], ss);
        if (ovl) {
          cudaEventRecord(xev[2 * k + 1], st2);
          last_l = xev[2 * k + 1];
        }
        split_rhs_kernel<Mech, GM><<<grhs, blk, 0, st>>>(b, it);
        if (events) cudaEventRecord(ev[4], st);
        n += 4;
      }
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      // live slots after the last K_ctl of the batch (iteration it - 1)
      if ((e = cudaMemcpyAsync(h_live, &b.live[(it - 1) & 1], sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               st)) != cudaSuccess)
        return e;
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
      if (ovl && (e = cudaStreamSynchronize(st2)) != cudaSuccess) return e;
      for (int j = 0; events && j < k; ++j) {
        cudaEvent_t* ev = events + j * (SPLIT_PHASES + 2);
        // phases: ctl ev0->ev1, jac (ev1 or ev5 on st2)->ev2, lu ev2->ev3, rhs (ev3 or ev1)->ev4
        const cudaEvent_t from[SPLIT_PHASES] = {ev[0], ovl ? ev[5] : ev[1], ev[2], ovl ? ev[1] : ev[3]};
        const cudaEvent_t to[SPLIT_PHASES] = {ev[1], ev[2], ev[3], ev[4]};
        for (int i = 0; i < SPLIT_PHASES; ++i) {
          float ms = 0.f;
          if (cudaEventElapsedTime(&ms, from[i], to[i]) == cudaSuccess) phase_ms[i] += ms;
        }
      }
      if (*h_live == 0) break;
    }
    *launches = n;
    return cudaSuccess;
  }
};

// LU diagnostic: the SPLIT path's own factor/solve routines on identical inputs
// (oct_factor, 8 lanes per cell, as K_lu; the record layout of K_lu; the
// thread-level substitutions of K_ctl's Newton solve, lurec_substitute).
// M[(i n + j) N + c] in, LAPACK getrf factors out (rows in pivoted order);
// piv: getrf swap indices derived from the row permutation; b: solution.
template <int NN>
__global__ void __launch_bounds__(128) split_lu_diag_kernel(long long N, double* M, int* piv, double* b, int* info,
                                                            double* rec) {
  constexpr int R = (NN + OCT - 1) / OCT, LUREC = (NN * NN + NN + (NN + 1) / 2 + 3) / 4 * 4;
  constexpr int LU_INVD = NN * NN, LU_PERM = NN * NN + NN;
  const int lane = threadIdx.x & 31, gl = lane & (OCT - 1);
  const unsigned gmask = 0xffu << (lane & ~(OCT - 1));
  const long long c = ((long long)blockIdx.x * 128 + threadIdx.x) / OCT;
  if (c >= N) return;                         // whole groups exit together (N is per group)
  double* lu = rec + c * LUREC;
  double a[R][NN];
#pragma unroll
  for (int s = 0; s < R; ++s) {
    const int r = gl + OCT * s;
#pragma unroll
    for (int j = 0; j < NN; ++j) a[s][j] = (r < NN) ? M[((long long)r * NN + j) * N + c] : 0.0;
  }
  int pos[R];
  double dinv[R];
  const int inf = oct_factor<NN>(gmask, gl, a, pos, dinv);
  if (!inf) {
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const int r = gl + OCT * s;
      if (r < NN) {
#pragma unroll
        for (int j = 0; j < NN; ++j) lu[j * NN + pos[s]] = a[s][j];
        lu[LU_INVD + pos[s]] = dinv[s];
        reinterpret_cast<int*>(lu + LU_PERM)[pos[s]] = r;
      }
    }
  }
  __syncwarp(gmask);
  if (gl != 0) return;
  info[c] = inf;
  if (inf) return;
  const int* perm = reinterpret_cast<const int*>(lu + LU_PERM);
  double x[NN];
#pragma unroll
  for (int i = 0; i < NN; ++i) x[i] = b[(long long)perm[i] * N + c];
  lurec_substitute<NN>(lu, x);
  for (int i = 0; i < NN; ++i) {
    b[(long long)i * N + c] = x[i];
    for (int j = 0; j < NN; ++j) M[((long long)i * NN + j) * N + c] = lu[j * NN + i];
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

size_t split_lu_rec_doubles(int n) { return (size_t)((n * n + n + (n + 1) / 2 + 3) / 4 * 4); }

cudaError_t split_geometry(int mech, int device, SplitGeom* gm) {
  switch (mech) {
    case BDFB_MODEL_MECH_H2: return KH2::geometry(device, gm);
    case BDFB_MODEL_MECH_DRM19: return KDRM::geometry(device, gm);
  }
  return cudaErrorInvalidValue;
}

cudaError_t split_integrate(int mech, const Opts& o, double* y, const double* fext, const double* aux,
                            const double* atol, const SplitBufs& sb, const SplitGeom& gm, unsigned long long* counter,
                            Agg* agg, const CellStatsPtrs& cs, unsigned long long* h_live, int batch,
                            cudaStream_t st, int* launches, cudaEvent_t* events, double* phase_ms, cudaStream_t st2,
                            cudaEvent_t* xev) {
  switch (mech) {
    case BDFB_MODEL_MECH_H2:
      return KH2::run(o, y, fext, aux, atol, sb, gm, counter, agg, cs, h_live, batch, st, launches, events,
                       phase_ms, st2, xev);
    case BDFB_MODEL_MECH_DRM19:
      return KDRM::run(o, y, fext, aux, atol, sb, gm, counter, agg, cs, h_live, batch, st, launches, events,
                        phase_ms, st2, xev);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bdfb
