// split_run.cuh -- host side of the SPLIT per-cell integrator (bdf_split.cuh): slot pool
// geometry and the host loop that enqueues the kernels of a trip, for one mechanism and one
// linear solver (LS_DENSE: K_ctl, K_jac, K_lu, K_rhs; LS_DIAG / LS_GMRES: K_ctl, K_rhs).
// Included by split.cu (dense) and split_mf.cu (matrix-free solvers).
#pragma once
#include <cuda_runtime.h>
#include <stdlib.h>

#include "bdf_split.cuh"
#include "split_api.h"
#include "split_big.cuh"
#include "erk_split.cuh"

namespace bdfb {
namespace {

template <class Mech, class GM, int LS = LS_DENSE>
struct SplitK {
  using SP = Split<Mech, GM, LS>;
  static constexpr size_t ctl_smem() {
    return BDFB_SPLIT_TS_SMEM ? sizeof(double) * (size_t)TS_STRIDE * BDFB_SPLIT_CTL_BLOCK : 0;
  }
  static constexpr bool BIG = Mech::N > 32;   // split_big.cuh setup kernels (lanes Jacobian, register-row LU)
  // two-pass generated Jacobian (split_jac_part/sum/p2_kernel; BDFB_SPLIT_JAC2=0: the group/lanes one)
  static constexpr bool JAC2 = LS == LS_DENSE;
  static constexpr size_t jac_smem() {
    if constexpr (BIG) {
      return sizeof(double) * (size_t)JacLanesSmem<Mech>::PER_WARP * JL_WARPS;
    } else {
      return sizeof(double) * (size_t)(GM::SG + GM::JG + GM::N * (GM::N | 1)) * (BDFB_SPLIT_BLOCK / GM::G);
    }
  }

  static cudaError_t geometry(int device, SplitGeom* gm) {
    cudaError_t e;
    const int sm = (int)ctl_smem();
    if ((e = cudaFuncSetAttribute(split_ctl_kernel<Mech, GM, LS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  sm > 110 * 1024 ? sm : 110 * 1024)) != cudaSuccess)
      return e;
    int nsm = 0, pr = 0;
    if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess) return e;
    if ((e = split_rhs_occupancy<Mech, GM, LS>(&pr)) != cudaSuccess) return e;
    if (pr < 1) return cudaErrorInvalidConfiguration;
    if constexpr (BIG) {
      if (LS == LS_DENSE && jac_smem() > 48 * 1024 &&
          (e = cudaFuncSetAttribute(split_jac_lanes_kernel<Mech, GM, LS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)jac_smem())) != cudaSuccess)
        return e;
    } else {
      if (LS == LS_DENSE && jac_smem() > 48 * 1024 &&
          (e = cudaFuncSetAttribute(split_jac_kernel<Mech, GM, LS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)jac_smem())) != cudaSuccess)
        return e;
    }
    gm->rhs_grid = nsm * pr;
    gm->setup_grid = nsm * 8;
    gm->vec_doubles = SP::D;
    gm->ts_doubles = TS_STRIDE;
    gm->jrec = LS == LS_DENSE ? SP::JREC : 0;   // no J / LU records for the matrix-free solvers
    gm->lurec = LS == LS_DENSE ? SP::LUREC : 0;
    if constexpr (JAC2) gm->jscr = jac_scr_doubles<Mech>();
    else gm->jscr = 0;
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
    if constexpr (!BIG) {   // K_lu: a persistent grid of exactly the resident blocks (no partial last wave)
      static int lu_res = -1;
      if (lu_res < 0) {
        int per = 0, nsm = gm.setup_grid / 8;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, split_lu_kernel<Mech, GM, LS>, blk, 0) != cudaSuccess ||
            per < 1)
          per = 2;
        lu_res = per * nsm;
      }
      if (glu > (unsigned)lu_res) glu = (unsigned)lu_res;
    }
    unsigned grhs = (unsigned)gm.rhs_grid;
    if (grhs > gs) grhs = gs;
    if (const char* g = getenv("BDFB_SPLIT_RHS_FULLGRID"))   // experiments: one thread per slot
      if (atoi(g) == 1) grhs = gs;
    size_t sm = ctl_smem();
    if (const char* pad = getenv("BDFB_SPLIT_CTL_SMEM")) {  // experiments: cap the resident K_ctl blocks
      const size_t want = (size_t)strtoul(pad, nullptr, 10);
      if (want > sm) sm = want;
    }
    split_init_kernel<Mech, GM, LS><<<gs, blk, 0, st>>>(b);
    bool jac_tpc = false;   // BDFB_SPLIT_JAC_TPC=1: thread-per-entry generated Jacobian (measurement)
    if (const char* jt = getenv("BDFB_SPLIT_JAC_TPC")) jac_tpc = atoi(jt) == 1;
    bool jac2 = true;       // BDFB_SPLIT_JAC2=0: the group (lanes) Jacobian instead of the two-pass generated one
    if (const char* j2 = getenv("BDFB_SPLIT_JAC2")) jac2 = atoi(j2) != 0;
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
        if constexpr (LS == LS_ERK)
          erk_ctl_kernel<Mech, GM><<<gs, blk, 0, st>>>(o, b, it, y, fext, aux, atol, counter, agg, cs);
        else
          split_ctl_kernel<Mech, GM, LS><<<gctl, BDFB_SPLIT_CTL_BLOCK, sm, st>>>(o, b, it, y, fext, aux, atol, counter,
                                                                           agg, cs);
#if BDFB_SPLIT_INIT_KERNEL
        split_init_cells_kernel<Mech, GM, LS><<<ginit, blk, 0, st>>>(o, b, it, y, fext, aux, atol, counter, agg, cs);
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
        if constexpr (LS == LS_DENSE && BIG) {   // n > 32: two-pass generated Jacobian, or the lanes one
          if (BDFB_SPLIT_JAC_PARTS && jac2 && b.jscr) {
            split_jac_part_kernel<Mech, GM, LS><<<(unsigned)gm.setup_grid, blk, 0, ss>>>(b, it);
            split_jac_sum_kernel<Mech, GM, LS><<<(unsigned)gm.setup_grid, blk, 0, ss>>>(b, it);
            split_jac_p2_kernel<Mech, GM, LS><<<(unsigned)gm.setup_grid, blk, 0, ss>>>(b, it);
            n += 2;
          } else {
            const unsigned gj = (unsigned)gm.setup_grid;
            split_jac_lanes_kernel<Mech, GM, LS><<<gj, 32 * JL_WARPS, jac_smem(), ss>>>(b, it);
          }
        } else if constexpr (LS == LS_DENSE) {   // the matrix-free linear solvers have no setup kernels
          if (b.jac_dq)
            split_dqjac_kernel<Mech, GM, LS><<<gdq, blk, 0, ss>>>(b, it);
          else if (jac_tpc)
            split_jac_tpc_kernel<Mech, GM, LS><<<(unsigned)gm.rhs_grid, blk, 0, ss>>>(b, it);
          else if (JAC2 && jac2 && b.jscr) {
            if constexpr (JAC2) {
              if (BDFB_SPLIT_JAC_PARTS) {
                split_jac_part_kernel<Mech, GM, LS><<<(unsigned)gm.setup_grid, blk, 0, ss>>>(b, it);
                split_jac_sum_kernel<Mech, GM, LS><<<(unsigned)gm.setup_grid, blk, 0, ss>>>(b, it);
                ++n;
              } else {
                split_jac_p1_kernel<Mech, GM, LS><<<(unsigned)gm.setup_grid, blk, 0, ss>>>(b, it);
              }
              split_jac_p2_kernel<Mech, GM, LS><<<(unsigned)gm.setup_grid, blk, 0, ss>>>(b, it);
              ++n;
            }
          } else
            split_jac_kernel<Mech, GM, LS><<<gjac, blk, jac_smem(), ss>>>(b, it);
        }
        if (events) cudaEventRecord(ev[2], ss);
        if constexpr (LS == LS_DENSE && BIG) {
          // two 192-thread blocks per SM (setup_grid = 8 per SM), grid-stride over the setup list
          split_lu_rows_kernel<Mech, GM, LS><<<(unsigned)(gm.setup_grid / 8 * LUR<Mech::N>::BPS), LUR<Mech::N>::T, 0,
                                                ss>>>(b, it);
        } else if constexpr (LS == LS_DENSE) {
          split_lu_kernel<Mech, GM, LS><<<glu, blk, 0, ss>>>(b, it);
        }
        if (events) cudaEventRecord(ev[3], ss);
        if (ovl) {
          cudaEventRecord(xev[2 * k + 1], st2);
          last_l = xev[2 * k + 1];
        }
        split_rhs_run<Mech, GM, LS>(grhs, st, b, it);
        if (events) cudaEventRecord(ev[4], st);
        n += (LS == LS_DENSE) ? 4 : 2;
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

}  // namespace
}  // namespace bdfb
