// erk.cu -- explicit adaptive Runge-Kutta integration of every cell (the paper's
// "fourth-order explicit method" from ARKODE), B200 / sm_100a; a translation unit of libbdfb.so.
//
// Method (reading R30; independent of oracle/erk.c, which restates it for the CPU): the
// Zonneveld 5-stage 4(3) pair, c = (0, 1/2, 1/2, 1, 3/4), a21 = a32 = 1/2, a43 = 1,
// a5j = (5/32, 7/32, 13/32, -1/32), b = (1/6, 1/3, 1/3, 1/6, 0), e = b - b^ = (2/3, -2, -2, -2, 16/3);
// the WRMS error test of Eq. 3 with the embedded estimate (accept iff ||h sum e_j k_j|| <= 1);
// eta = 0.9 / dsm^(1/4) capped at 1e4 (first step), 10, or 1 after a failure; rejection eta >= 0.1; the
// Hairer-Wanner initial step with the R25 fifth root; a recoverable RHS failure in a stage cuts h by 1/4.
//
// GPU organisation: ONE CELL PER THREAD in a persistent grid that pulls cells from the device work
// counter.  Each thread is a flat state machine whose only RHS call site is shared by every phase
// (f(t0, y0), the initial-step probe, k1 after an accepted step, stages 2..5), so a warp's lanes -- at
// different steps of different cells -- always evaluate the generated straight-line RHS
// (gen/tpc_<mech>.cuh) together, and a block barrier per trip keeps the block's 12 warps in the same
// stretch of that code (one block per SM): full warps on the FP64 pipe, no algebraic solver.
// The cell's vectors (y, F, k1..k5, weights: 8n doubles) live in a per-thread workspace sized for the
// resident grid, element-major across threads (one coalesced 256-byte line pair per warp access; 80 MB
// for DRM19 on 148 SMs, L2-resident).
#include <cuda_runtime.h>
#include <math.h>

#include "../../include/bdfb.h"
#include "bdf_cell.cuh"
#include "erk_api.h"
#include "gen/tpc_drm19_class.cuh"
#include "gen/tpc_h2_lidryer.cuh"
#include "gen/tpc_gri53_class.cuh"

namespace bdfb {
namespace {

// one block of 12 warps per SM, block-synchronous RHS calls: the generated RHS is ~10K instructions of
// straight-line SASS; warps at different places in it thrash the instruction cache (ncu, 128-thread
// blocks without the barrier: 38 of 49 stall cycles per issue "no instruction", IPC 0.23)
#ifndef BDFB_ERK_BLOCK
#define BDFB_ERK_BLOCK 384
#endif
#ifndef BDFB_ERK_MINB
#define BDFB_ERK_MINB 1
#endif

constexpr double ERK_SAFETY = 0.9, ERK_ETAMX1 = 1e4, ERK_ETAMX = 10.0, ERK_ETAMIN = 0.1, ERK_ETACF = 0.25;
constexpr int ERK_MXNEF = 7, ERK_MXNCF = 10;
// tableau rows: stage s (1..4, i.e. k2..k5) uses A[s][j] for j < s
__constant__ double kErkA[5][4] = {{0, 0, 0, 0},
                                   {0.5, 0, 0, 0},
                                   {0, 0.5, 0, 0},
                                   {0, 0, 1.0, 0},
                                   {5.0 / 32.0, 7.0 / 32.0, 13.0 / 32.0, -1.0 / 32.0}};

// request phases: what the next RHS value is
enum : int { R_F0 = 0, R_H0 = 1, R_K1 = 2, R_S2 = 3, R_S5 = 6, R_NONE = 7 };

template <int N>
struct EW {   // per-thread workspace: element e at w[e * S]
  double* w;
  long long S;
  __device__ __forceinline__ double& at(int e) const { return w[(long long)e * S]; }
  __device__ __forceinline__ double& y(int i) const { return at(i); }
  __device__ __forceinline__ double& F(int i) const { return at(N + i); }
  __device__ __forceinline__ double& k(int s, int i) const { return at(2 * N + s * N + i); }
  __device__ __forceinline__ double& ewt(int i) const { return at(7 * N + i); }
};

template <int N>
__device__ __forceinline__ double wnorm_k(const EW<N>& w, int s) {   // ||k_s||_WRMS, sequential order
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double p = w.k(s, i) * w.ewt(i);
    acc = acc + p * p;
  }
  return sqrt(acc / (double)N);
}

// the request of a phase, the generated RHS and f + F into its k slot (k1 for f(t0, y0) and f(tn, yn), k2 for
// the initial-step probe, k_s for stage s), out of line: the register-hungry RHS gets its own allocation and
// the state machine around it stays light
// e^{-g/RT} and its reciprocals of the generated RHS in shared memory (rhs_sm; 2K doubles per thread) when they
// fit next to the scalar state, else in registers
template <class Mech>
__host__ __device__ constexpr bool erk_sm() {
  return 2 * Mech::K * BDFB_ERK_BLOCK * 8 + 15 * 8 * BDFB_ERK_BLOCK <= 200 * 1024;
}
template <class Mech>
__host__ __device__ constexpr size_t erk_sm_bytes() {
  return erk_sm<Mech>() ? sizeof(double) * 2 * Mech::K * BDFB_ERK_BLOCK : 0;
}

template <class Mech>
__device__ __noinline__ int erk_eval(const EW<Mech::N> w, int phase, double hs, double h0, double rho) {
  constexpr int N = Mech::N;
  double yv[N], fv[N];
  int dst = 0;
  if (phase == R_F0 || phase == R_K1) {
#pragma unroll
    for (int i = 0; i < N; ++i) yv[i] = w.y(i);
  } else if (phase == R_H0) {
    dst = 1;
#pragma unroll
    for (int i = 0; i < N; ++i) yv[i] = h0 * w.k(0, i) + w.y(i);
  } else {                       // stage s = phase - R_K1 (1..4): y + h sum_{j<s, a_sj != 0} a_sj k_j
    const int st = phase - R_K1;
    dst = st;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
      bool first = true;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double a = kErkA[st][j];
        if (j < st && a != 0.0) {
          const double tj = a * w.k(j, i);
          acc = first ? tj : acc + tj;
          first = false;
        }
      }
      yv[i] = hs * acc + w.y(i);
    }
  }
  int rv;
  if constexpr (erk_sm<Mech>()) {
    extern __shared__ double esm[];
    rv = Mech::template rhs_sm<BDFB_ERK_BLOCK>(yv, rho, fv, esm + threadIdx.x);
  } else {
    rv = Mech::rhs(yv, rho, fv);
  }
#pragma unroll
  for (int i = 0; i < N; ++i) w.k(dst, i) = fv[i] + w.F(i);
  return rv;
}

struct ES {   // scalar state of a thread's cell (15 doubles)
  double rho, t, h, hs, h0, d1, etamax, hlast;
  long long cell;
  int nst, nfe, netf, ncfn, nef, ncf, status, last, phase, pad[3];
};
static_assert(sizeof(ES) == 15 * 8, "odd stride in doubles");

template <class Mech>
__global__ void __launch_bounds__(BDFB_ERK_BLOCK, BDFB_ERK_MINB)
    erk_kernel(Opts o, double* y, const double* fext, const double* aux, const double* atol, double* ws,
               unsigned long long* counter, Agg* agg, CellStatsPtrs cs) {
  constexpr int N = Mech::N;
  const long long S = (long long)gridDim.x * BDFB_ERK_BLOCK;
  const EW<N> w{ws + (long long)blockIdx.x * BDFB_ERK_BLOCK + threadIdx.x, S};
  auto idx = [&](long long c, int k) { return o.layout == 0 ? (long long)k * o.ncells + c : c * (long long)N + k; };
  const double B[4] = {1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0};
  const double E[5] = {2.0 / 3.0, -2.0, -2.0, -2.0, 16.0 / 3.0};

  // the cell's scalar state lives in shared memory (an odd number of doubles per thread: conflict-free), so
  // that only addresses stay live in registers across the register-hungry generated RHS
  __shared__ ES sst[BDFB_ERK_BLOCK];
  ES& es = sst[threadIdx.x];
  long long& cell = es.cell;
  double &rho = es.rho, &t = es.t, &h = es.h, &hs = es.hs, &h0 = es.h0, &d1 = es.d1, &etamax = es.etamax,
         &hlast = es.hlast;
  int &nst = es.nst, &nfe = es.nfe, &netf = es.netf, &ncfn = es.ncfn, &nef = es.nef, &ncf = es.ncf,
      &status = es.status, &last = es.last, &phase = es.phase;
  cell = -1;
  etamax = ERK_ETAMX1;
  nef = ncf = last = 0;
  phase = R_NONE;
  bool alive = true;
  for (;;) {
    if (alive && phase == R_NONE) {   // load the next cell
      const long long c = (long long)atomicAdd(counter, 1ull);
      if (c >= o.ncells) alive = false;
      else cell = c;
    }
    // the block's warps enter the RHS together (instruction-cache locality); the block retires with its last cell
    if (!__syncthreads_or(alive)) break;
    if (!alive) continue;
    if (phase == R_NONE) {
      const long long c = cell;
      rho = aux ? aux[c] : 0.0;
      bool bad = !isfinite(rho);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double y0 = y[idx(c, i)];
        const double fe = fext ? fext[idx(c, i)] : 0.0;
        if (!isfinite(y0) || !isfinite(fe)) bad = true;
        w.y(i) = y0;
        w.F(i) = fe;
        w.ewt(i) = 1.0 / (o.rtol * fabs(y0) + atol[i]);
      }
      nst = nfe = netf = ncfn = 0;
      t = o.t0;
      h = hlast = 0.0;
      status = bad ? ST_NONFINITE : ST_OK;
      phase = bad ? -1 : R_F0;
    }
    if (phase >= 0) {
      // ---- the single RHS call site: build the request vector of this phase
      const int rv = erk_eval<Mech>(w, phase, hs, h0, rho);
      nfe++;
      // ---- consume
      if (phase == R_F0 || phase == R_K1) {
        if (rv) {
          status = ST_RHS_FAIL;
          phase = -1;
        } else {
#pragma unroll
          if (phase == R_F0) {
            if (o.h0 != 0.0) {
              h = o.h0;
              phase = -2;   // start stepping
            } else {         // Hairer-Wanner starting step: the probe f(t0 + h0, y0 + h0 f0)
              double a0 = 0.0;
#pragma unroll
              for (int i = 0; i < N; ++i) {
                const double p = w.y(i) * w.ewt(i);
                a0 = a0 + p * p;
              }
              const double d0 = sqrt(a0 / (double)N);
              d1 = wnorm_k<N>(w, 0);
              h0 = (d0 < 1e-5 || d1 < 1e-5) ? 1e-6 : 0.01 * (d0 / d1);
              if (h0 > o.tf - o.t0) h0 = o.tf - o.t0;
              phase = R_H0;
            }
          } else {
            phase = -3;      // after an accepted step: the mxstep check, then a new attempt
          }
        }
      } else if (phase == R_H0) {
        if (rv) {
          h = h0;
        } else {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            const double d = w.k(1, i) - w.k(0, i);
            const double p = d * w.ewt(i);
            acc = acc + p * p;
          }
          const double d2 = sqrt(acc / (double)N) / h0;
          const double dm = fmax(d1, d2);
          const double h1 = (dm <= 1e-15) ? fmax(1e-6, h0 * 1e-3) : root_l(0.01 / dm, 5);
          h = fmin(100.0 * h0, h1);
        }
        phase = -2;
      } else {                 // stage s of the attempt
        const int st = phase - R_K1;
        if (rv) {              // recoverable RHS failure: cut h, retry the step (k1 kept)
          ncfn++;
          if (++ncf == ERK_MXNCF) {
            status = ST_RHS_FAIL;
            phase = -1;
          } else {
            h = h * ERK_ETACF;
            etamax = 1.0;
            phase = -4;
          }
        } else {
          if (phase < R_S5) {
            phase++;
          } else {             // all five stages: solution, estimate, error test
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
              double e = E[0] * w.k(0, i);
#pragma unroll
              for (int j = 1; j < 5; ++j) e = e + E[j] * w.k(j, i);
              const double p = (hs * e) * w.ewt(i);
              acc = acc + p * p;
            }
            const double dsm = sqrt(acc / (double)N);
            if (dsm <= 1.0) {  // accept
              nst++;
#pragma unroll
              for (int i = 0; i < N; ++i) {
                double sb = B[0] * w.k(0, i);
#pragma unroll
                for (int j = 1; j < 4; ++j) sb = sb + B[j] * w.k(j, i);
                w.y(i) = hs * sb + w.y(i);
              }
              t = last ? o.tf : t + hs;
              hlast = hs;
              if (last) {
                phase = -1;
              } else {
                double eta = (dsm == 0.0) ? etamax : ERK_SAFETY / sqrt(sqrt(dsm));
                eta = fmin(eta, etamax);
                if (o.hmax > 0.0) eta = fmin(eta, o.hmax / fabs(hs));
                h = hs * eta;
                etamax = ERK_ETAMX;
#pragma unroll
                for (int i = 0; i < N; ++i) w.ewt(i) = 1.0 / (o.rtol * fabs(w.y(i)) + atol[i]);
                phase = R_K1;
              }
            } else {           // reject
              netf++;
              if (++nef == ERK_MXNEF || fabs(hs) <= o.hmin * (1.0 + UROUND)) {
                status = ST_ERR_FAILURE;
                phase = -1;
              } else {
                double eta = fmax(ERK_ETAMIN, ERK_SAFETY / sqrt(sqrt(dsm)));
                if (o.hmin > 0.0) eta = fmax(eta, o.hmin / fabs(hs));
                h = hs * eta;
                etamax = 1.0;
                if (t + h == t) {
                  status = ST_ERR_FAILURE;
                  phase = -1;
                } else {
                  phase = -4;
                }
              }
            }
          }
        }
      }
    }
    // ---- control transitions without an RHS value
    if (phase == -2) {         // first step: clip h0, etamax
      if (h > o.tf - o.t0) h = o.tf - o.t0;
      if (o.hmax > 0.0 && h > o.hmax) h = o.hmax;
      etamax = ERK_ETAMX1;
      phase = -3;
    }
    if (phase == -3) {         // top of a step: mxstep, then a fresh attempt
      if (nst >= o.mxstep) {
        status = ST_TOO_MUCH_WORK;
        phase = -1;
      } else {
        nef = 0;
        ncf = 0;
        phase = -4;
      }
    }
    if (phase == -4) {         // attempt: clip to tf, stage 2 request (k1 at hand)
      last = 0;
      hs = h;
      if ((t + hs - o.tf) >= 0.0) {
        hs = o.tf - t;
        last = 1;
      }
      h = hs;
      phase = R_S2;
    }
    if (phase == -1) {         // store the cell
      const long long c = cell;
      if (status != ST_NONFINITE) {
#pragma unroll
        for (int i = 0; i < N; ++i) y[idx(c, i)] = w.y(i);
      }
      if (cs.status) cs.status[c] = status;
      if (cs.nst) cs.nst[c] = nst;
      if (cs.nfe) cs.nfe[c] = nfe;
      if (cs.nje) cs.nje[c] = 0;
      if (cs.nsetups) cs.nsetups[c] = 0;
      if (cs.nni) cs.nni[c] = 0;
      if (cs.netf) cs.netf[c] = netf;
      if (cs.ncfn) cs.ncfn[c] = ncfn;
      if (cs.q_last) cs.q_last[c] = 4;
      if (cs.h_last) cs.h_last[c] = hlast;
      if (cs.t_reached) cs.t_reached[c] = t;
      atomicAdd(&agg->n_failed, (unsigned long long)(status != ST_OK));
      atomicAdd(&agg->nst, (unsigned long long)nst);
      atomicAdd(&agg->nfe, (unsigned long long)nfe);
      atomicAdd(&agg->netf, (unsigned long long)netf);
      atomicAdd(&agg->ncfn, (unsigned long long)ncfn);
      atomicMax(&agg->nst_max, (unsigned long long)nst);
      atomicMax(&agg->nfe_max, (unsigned long long)nfe);
      atomicAdd(&agg->cells_done, 1ull);
      phase = R_NONE;
    }
  }
}

template <class Mech>
cudaError_t geometry(int device, long long ncells, long long* threads, long long* dpt) {
  int nsm = 0, pr = 0;
  cudaError_t e;
  if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess) return e;
  if (erk_sm_bytes<Mech>() > 48 * 1024 &&
      (e = cudaFuncSetAttribute(erk_kernel<Mech>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)erk_sm_bytes<Mech>())) != cudaSuccess)
    return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pr, erk_kernel<Mech>, BDFB_ERK_BLOCK,
                                                         erk_sm_bytes<Mech>())) != cudaSuccess)
    return e;
  if (pr < 1) return cudaErrorInvalidConfiguration;
  long long blocks = (long long)nsm * pr;
  const long long need = (ncells + BDFB_ERK_BLOCK - 1) / BDFB_ERK_BLOCK;
  if (blocks > need) blocks = need;
  *threads = blocks * BDFB_ERK_BLOCK;
  *dpt = 8 * Mech::N;
  return cudaSuccess;
}

}  // namespace

cudaError_t erk_geometry(int mech, int device, long long ncells, long long* threads, long long* doubles_per_thread) {
  switch (mech) {
    case BDFB_MODEL_MECH_H2: return geometry<Tpc_h2_lidryer>(device, ncells, threads, doubles_per_thread);
    case BDFB_MODEL_MECH_DRM19: return geometry<Tpc_drm19_class>(device, ncells, threads, doubles_per_thread);
    case BDFB_MODEL_MECH_GRI53: return geometry<Tpc_gri53_class>(device, ncells, threads, doubles_per_thread);
  }
  return cudaErrorInvalidValue;
}

cudaError_t erk_integrate(int mech, const Opts& o, double* y, const double* fext, const double* aux,
                          const double* atol, double* ws, long long threads, unsigned long long* counter, Agg* agg,
                          const CellStatsPtrs& cs, cudaStream_t st) {
  const unsigned grid = (unsigned)(threads / BDFB_ERK_BLOCK);
  switch (mech) {
    case BDFB_MODEL_MECH_H2:
      erk_kernel<Tpc_h2_lidryer><<<grid, BDFB_ERK_BLOCK, erk_sm_bytes<Tpc_h2_lidryer>(), st>>>(o, y, fext, aux, atol, ws, counter, agg, cs);
      break;
    case BDFB_MODEL_MECH_DRM19:
      erk_kernel<Tpc_drm19_class><<<grid, BDFB_ERK_BLOCK, erk_sm_bytes<Tpc_drm19_class>(), st>>>(o, y, fext, aux, atol, ws, counter, agg, cs);
      break;
    case BDFB_MODEL_MECH_GRI53:
      erk_kernel<Tpc_gri53_class><<<grid, BDFB_ERK_BLOCK, erk_sm_bytes<Tpc_gri53_class>(), st>>>(o, y, fext, aux, atol, ws, counter, agg, cs);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace bdfb
