// erk_split.cuh -- the explicit adaptive ERK (row f4; erk.cu's method, reading R30) in the SPLIT organisation:
// the slot pool of bdf_split.cuh, a light control kernel (K_erk: consume the RHS value of the slot's request,
// the step-size control, the next stage vector) and the SPLIT RHS kernel (K_rhs, the generated RHS with its
// e^{-g/RT} in shared memory, 30% of FP64 on full warps).  Versus the persistent erk_kernel (RHS in line,
// block-synchronous trips) the RHS no longer shares registers, occupancy and barriers with the control.
//
// Slot record mapping (the dense-BDF records, reinterpreted; LS_ERK has no J / LU):
//   VEC  zn[0] = y, zn[1..5] = k1..k5, ewt, fext = F, yq = request, fr = f(yq) + F
//   TS   tn = t, h, hprime = the attempt's h (hs), eta = h0 (initial-step probe), saved_t = d1, etamax,
//        hscale = h of the last accepted step; nst, nfe, netf, ncfn; nef, ncf, status; m = the ERK phase,
//        flag = last; phase = PH_NRES while a request is pending (the K_rhs predicate), PH_DONE when empty.
// Operations and their order are erk.cu's (and the oracle's orc_integrate_erk).
#pragma once
#include "bdf_split.cuh"

namespace bdfb {

constexpr int LS_ERK = 3;   // the "linear solver" slot of the SPLIT templates: the ERK organisation

// ERK phases (TS.m): the RHS value in fr answers this request
enum : int { E_F0 = 0, E_H0 = 1, E_K1 = 2, E_S2 = 3, E_S5 = 6 };

template <class Mech, class GM>
struct ErkSplit {
  using SP = Split<Mech, GM, LS_ERK>;
  using W = typename SP::W;
  static constexpr int N = Mech::N;
  static constexpr double SAFETY = 0.9, ETAMX1 = 1e4, ETAMX = 10.0, ETAMIN = 0.1, ETACF = 0.25;
  static constexpr int MXNEF = 7, MXNCF = 10;
  __device__ static double& y(const W& w, int i) { return w.zn(0, i); }
  __device__ static double& k(const W& w, int s, int i) { return w.zn(1 + s, i); }

  // the request vector of phase ph into yq (stage s: y + h sum_{j<s, a_sj != 0} a_sj k_j)
  __device__ static void request(TS& s, const W& w, int ph) {
    const double A[5][4] = {{0, 0, 0, 0}, {0.5, 0, 0, 0}, {0, 0.5, 0, 0}, {0, 0, 1.0, 0},
                            {5.0 / 32.0, 7.0 / 32.0, 13.0 / 32.0, -1.0 / 32.0}};
    if (ph == E_F0 || ph == E_K1) {
#pragma unroll
      for (int i = 0; i < N; ++i) w.yq(i) = y(w, i);
    } else if (ph == E_H0) {
#pragma unroll
      for (int i = 0; i < N; ++i) w.yq(i) = s.eta * k(w, 0, i) + y(w, i);
    } else {
      const int st = ph - E_K1;
      const double hs = s.hprime;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double acc = 0.0;
        bool first = true;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double a = 0.0;
#pragma unroll
          for (int r = 1; r < 5; ++r)
            if (r == st) a = A[r][j];
          if (j < st && a != 0.0) {
            const double tj = a * k(w, j, i);
            acc = first ? tj : acc + tj;
            first = false;
          }
        }
        w.yq(i) = hs * acc + y(w, i);
      }
    }
    s.m = (signed char)ph;
    s.phase = PH_NRES;
  }

  __device__ static void store(const Opts& o, TS& s, const W& w, double* yout, Agg& acc, const CellStatsPtrs& cs) {
    const long long c = s.cell;
    auto idx = [&](int kk) { return o.layout == 0 ? (long long)kk * o.ncells + c : c * (long long)N + kk; };
    if (s.status != ST_NONFINITE) {
#pragma unroll
      for (int i = 0; i < N; ++i) yout[idx(i)] = y(w, i);
    }
    if (cs.status) cs.status[c] = s.status;
    if (cs.nst) cs.nst[c] = s.nst;
    if (cs.nfe) cs.nfe[c] = s.nfe;
    if (cs.nje) cs.nje[c] = 0;
    if (cs.nsetups) cs.nsetups[c] = 0;
    if (cs.nni) cs.nni[c] = 0;
    if (cs.netf) cs.netf[c] = s.netf;
    if (cs.ncfn) cs.ncfn[c] = s.ncfn;
    if (cs.q_last) cs.q_last[c] = 4;
    if (cs.h_last) cs.h_last[c] = s.hscale;
    if (cs.t_reached) cs.t_reached[c] = s.tn;
    atomicAdd(&acc.n_failed, (unsigned long long)(s.status != ST_OK));
    atomicAdd(&acc.nst, (unsigned long long)s.nst);
    atomicAdd(&acc.nfe, (unsigned long long)s.nfe);
    atomicAdd(&acc.netf, (unsigned long long)s.netf);
    atomicAdd(&acc.ncfn, (unsigned long long)s.ncfn);
    atomicMax(&acc.nst_max, (unsigned long long)s.nst);
    atomicMax(&acc.nfe_max, (unsigned long long)s.nfe);
    atomicAdd(&acc.cells_done, 1ull);
    s.phase = PH_DONE;
  }

  // next cell from the device work counter (f(t0, y0) requested); false when the counter is exhausted
  __device__ static bool load(const Opts& o, TS& s, const W& w, double* yin, const double* fext, const double* aux,
                              const double* atol, unsigned long long* counter, Agg& acc, const CellStatsPtrs& cs) {
    for (;;) {
      const long long c = (long long)atomicAdd(counter, 1ull);
      if (c >= o.ncells) {
        s.phase = PH_DONE;
        return false;
      }
      auto idx = [&](int kk) { return o.layout == 0 ? (long long)kk * o.ncells + c : c * (long long)N + kk; };
      s.cell = c;
      s.aux = aux ? aux[c] : 0.0;
      bool bad = !isfinite(s.aux);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double y0 = yin[idx(i)];
        const double fe = fext ? fext[idx(i)] : 0.0;
        if (!isfinite(y0) || !isfinite(fe)) bad = true;
        y(w, i) = y0;
        w.fext(i) = fe;
        w.ewt(i) = 1.0 / (o.rtol * fabs(y0) + atol[i]);
      }
      s.nst = s.nfe = s.netf = s.ncfn = 0;
      s.tn = o.t0;
      s.h = s.hscale = 0.0;
      s.nef = s.ncf = 0;
      s.flag = 0;
      s.etamax = ETAMX1;
      if (bad) {
        s.status = ST_NONFINITE;
        store(o, s, w, yin, acc, cs);
        continue;
      }
      s.status = ST_OK;
      request(s, w, E_F0);
      return true;
    }
  }

  // one trip: consume the RHS value (rv, fr) of the pending request, control, the next request / store + load.
  // Returns true while the slot holds a cell with a pending request.
  __device__ static bool trip(const Opts& o, TS& s, const W& w, int rv, double* yio, const double* fext,
                              const double* aux, const double* atol, unsigned long long* counter, Agg& acc,
                              const CellStatsPtrs& cs) {
    const double B[4] = {1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0};
    const double E[5] = {2.0 / 3.0, -2.0, -2.0, -2.0, 16.0 / 3.0};
    const int ph = s.m;
    s.nfe++;
    int next = -9;             // -1 store, -2 first step, -3 step top, -4 attempt, else a request phase
    if (ph == E_F0 || ph == E_K1) {
      if (rv) {
        s.status = ST_RHS_FAIL;
        next = -1;
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) k(w, 0, i) = w.fr(i);
        if (ph == E_F0) {
          if (o.h0 != 0.0) {
            s.h = o.h0;
            next = -2;
          } else {
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
              const double p = y(w, i) * w.ewt(i);
              a0 = a0 + p * p;
            }
#pragma unroll
            for (int i = 0; i < N; ++i) {
              const double p = k(w, 0, i) * w.ewt(i);
              a1 = a1 + p * p;
            }
            const double d0 = sqrt(a0 / (double)N), d1 = sqrt(a1 / (double)N);
            s.saved_t = d1;
            double h0 = (d0 < 1e-5 || d1 < 1e-5) ? 1e-6 : 0.01 * (d0 / d1);
            if (h0 > o.tf - o.t0) h0 = o.tf - o.t0;
            s.eta = h0;
            next = E_H0;
          }
        } else {
          next = -3;
        }
      }
    } else if (ph == E_H0) {
      if (rv) {
        s.h = s.eta;
      } else {
        double acc2 = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double d = w.fr(i) - k(w, 0, i);
          const double p = d * w.ewt(i);
          acc2 = acc2 + p * p;
        }
        const double h0 = s.eta;
        const double d2 = sqrt(acc2 / (double)N) / h0;
        const double dm = fmax(s.saved_t, d2);
        const double h1 = (dm <= 1e-15) ? fmax(1e-6, h0 * 1e-3) : root_l(0.01 / dm, 5);
        s.h = fmin(100.0 * h0, h1);
      }
      next = -2;
    } else {                    // stage st of the attempt
      const int st = ph - E_K1;
      if (rv) {
        s.ncfn++;
        if (++s.ncf == MXNCF) {
          s.status = ST_RHS_FAIL;
          next = -1;
        } else {
          s.h = s.h * ETACF;
          s.etamax = 1.0;
          next = -4;
        }
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int r = 1; r < 5; ++r)
            if (r == st) k(w, r, i) = w.fr(i);
        if (ph < E_S5) {
          next = ph + 1;
        } else {
          const double hs = s.hprime;
          double acc2 = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double e = E[0] * k(w, 0, i);
#pragma unroll
            for (int j = 1; j < 5; ++j) e = e + E[j] * k(w, j, i);
            const double p = (hs * e) * w.ewt(i);
            acc2 = acc2 + p * p;
          }
          const double dsm = sqrt(acc2 / (double)N);
          if (dsm <= 1.0) {     // accept
            s.nst++;
#pragma unroll
            for (int i = 0; i < N; ++i) {
              double sb = B[0] * k(w, 0, i);
#pragma unroll
              for (int j = 1; j < 4; ++j) sb = sb + B[j] * k(w, j, i);
              y(w, i) = hs * sb + y(w, i);
            }
            s.tn = s.flag ? o.tf : s.tn + hs;
            s.hscale = hs;
            if (s.flag) {
              next = -1;
            } else {
              double eta = (dsm == 0.0) ? s.etamax : SAFETY / sqrt(sqrt(dsm));
              eta = fmin(eta, s.etamax);
              if (o.hmax > 0.0) eta = fmin(eta, o.hmax / fabs(hs));
              s.h = hs * eta;
              s.etamax = ETAMX;
#pragma unroll
              for (int i = 0; i < N; ++i) w.ewt(i) = 1.0 / (o.rtol * fabs(y(w, i)) + atol[i]);
              next = E_K1;
            }
          } else {              // reject
            s.netf++;
            if (++s.nef == MXNEF || fabs(hs) <= o.hmin * (1.0 + UROUND)) {
              s.status = ST_ERR_FAILURE;
              next = -1;
            } else {
              double eta = fmax(ETAMIN, SAFETY / sqrt(sqrt(dsm)));
              if (o.hmin > 0.0) eta = fmax(eta, o.hmin / fabs(hs));
              s.h = hs * eta;
              s.etamax = 1.0;
              if (s.tn + s.h == s.tn) {
                s.status = ST_ERR_FAILURE;
                next = -1;
              } else {
                next = -4;
              }
            }
          }
        }
      }
    }
    if (next == -2) {           // first step: clip h0, etamax
      if (s.h > o.tf - o.t0) s.h = o.tf - o.t0;
      if (o.hmax > 0.0 && s.h > o.hmax) s.h = o.hmax;
      s.etamax = ETAMX1;
      next = -3;
    }
    if (next == -3) {           // top of a step: mxstep, then a fresh attempt
      if (s.nst >= o.mxstep) {
        s.status = ST_TOO_MUCH_WORK;
        next = -1;
      } else {
        s.nef = 0;
        s.ncf = 0;
        next = -4;
      }
    }
    if (next == -4) {           // attempt: clip to tf, stage 2 request (k1 at hand)
      s.flag = 0;
      double hs = s.h;
      if ((s.tn + hs - o.tf) >= 0.0) {
        hs = o.tf - s.tn;
        s.flag = 1;
      }
      s.h = hs;
      s.hprime = hs;
      next = E_S2;
    }
    if (next == -1) {
      store(o, s, w, yio, acc, cs);
      return load(o, s, w, yio, fext, aux, atol, counter, acc, cs);
    }
    request(s, w, next);
    return true;
  }
};

// K_erk: one trip of every slot (thread per slot; the slot's TS record accessed in place, L1-cached)
template <class Mech, class GM>
__global__ void __launch_bounds__(BDFB_SPLIT_BLOCK) erk_ctl_kernel(Opts o, SplitBufs b, int it, double* y,
                                                                 const double* fext, const double* aux,
                                                                 const double* atol, unsigned long long* counter,
                                                                 Agg* agg, CellStatsPtrs cs) {
  using ES = ErkSplit<Mech, GM>;
  using SP = typename ES::SP;
  __shared__ Agg wacc[BDFB_SPLIT_BLOCK / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) wacc[warp] = Agg{};
  __syncwarp();
  if (blockIdx.x == 0 && threadIdx.x == 0) b.live[(it + 1) & 1] = 0;
  const long long slot = (long long)blockIdx.x * BDFB_SPLIT_BLOCK + threadIdx.x;
  bool live = false;
  if (slot < b.slots) {
    TS& s = *SP::ts(b, slot);
    const typename SP::W w = SP::ws(b, slot);
    if (s.phase == PH_DONE) {
      if (*reinterpret_cast<volatile unsigned long long*>(counter) < (unsigned long long)o.ncells)
        live = ES::load(o, s, w, y, fext, aux, atol, counter, wacc[warp], cs);
    } else {
      live = ES::trip(o, s, w, b.rv[slot], y, fext, aux, atol, counter, wacc[warp], cs);
    }
  }
  const unsigned bl = __ballot_sync(0xffffffffu, live);
  if (lane == 0 && bl) atomicAdd(&b.live[it & 1], (unsigned long long)__popc(bl));
  __syncwarp();
  if (lane == 0 && wacc[warp].cells_done) {
    const Agg& a = wacc[warp];
    atomicAdd(&agg->n_failed, a.n_failed);
    atomicAdd(&agg->nst, a.nst);
    atomicAdd(&agg->nfe, a.nfe);
    atomicAdd(&agg->netf, a.netf);
    atomicAdd(&agg->ncfn, a.ncfn);
    atomicMax(&agg->nst_max, a.nst_max);
    atomicMax(&agg->nfe_max, a.nfe_max);
    atomicAdd(&agg->cells_done, a.cells_done);
  }
}

}  // namespace bdfb
