// global_host.cuh -- host control loop of the global-norm mode (see
// global_mode.cuh).  The listing ("Global-norm variant")
// with every vector operation a device kernel over all cells and every norm a
// deterministic device reduction; with a communicator, the rank partials are
// exchanged with ncclAllGather and summed in rank order on every rank, so all
// ranks take identical decisions (one h, q for the whole multi-GPU batch).
#pragma once
#include <nccl.h>

#include <type_traits>
#include <vector>

#include "../../include/bdfb.h"
#include "global_lanes.cuh"
#include "global_mode.cuh"
#include "global_tpc.cuh"
#include "split_api.h"

namespace bdfb {

// n = 54 global-norm J: the generated two-pass Jacobian of the SPLIT path (default) or, with BDFB_GLOBAL_JAC2=0,
// the table-driven lanes model (gl_setup; 263 ns per cell vs ~50 ns, profiles/r2)
static inline bool gl_jac2() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BDFB_GLOBAL_JAC2");
    v = (e && atoi(e) == 0) ? 0 : 1;
  }
  return v == 1;
}

struct GlobalBuffers {           // allocated once (bdfb_create, GLOBAL_NORM mode)
  GVec v{};
  double *J = nullptr, *LU = nullptr, *invd = nullptr, *s = nullptr, *P = nullptr, *sum = nullptr, *gath = nullptr;
  int *pos = nullptr, *perm = nullptr, *flag = nullptr, *igath = nullptr;
  unsigned long long* ubuf = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  long long ncells_total = 0;
};

struct GlobalResult {
  int status;
  long long nst, nfe, nje, nsetups, nni, netf, ncfn;
  int q;
  double h, tn;
  long long launches;
};

// Tpc: the thread-per-cell mechanism type (gen/tpc_<mech>.cuh) whose kernels (global_tpc.cuh) do the RHS,
// setup and solve; void: the group kernels of global_mode.cuh
// lanes models (mech_lanes.cuh, any n): the kernels of global_lanes.cuh
template <class M, class = void>
struct IsLanes : std::false_type {};
template <class M>
struct IsLanes<M, std::void_t<decltype(M::LANES)>> : std::bool_constant<M::LANES> {};

// Tpc: the generated thread-per-cell RHS (and, for group models, setup and solve).  For the lanes model of
// C5 (n = 54) only its RHS is used (gt_rhs); J stays the table-driven lanes Jacobian, the LU is gl_lu.
template <class Model, class Tpc = void>
struct GlobalRunner {
  static constexpr bool TPC = !std::is_void<Tpc>::value;
  static constexpr bool LANES = IsLanes<Model>::value;
  using TM = typename std::conditional<TPC, Tpc, Model>::type;
  using P = typename Model::Params;
  static constexpr int QM = QMAX;
  GlobalBuffers& B;
  const Opts o;
  const P prm;
  cudaStream_t st;
  const int n;
  const long long N, M;
  const double* atol;
  const double* fext;
  const double* aux;
  long long launches = 0;
  // scalar state (the listing's)
  double tn = 0, h = 0, hscale = 0, hprime = 0, eta = 1, etamax = ETAMX1, saved_t = 0;
  double tau[QMAX + 2] = {0}, l[QMAX + 1] = {0}, tq[6] = {0};
  double rl1 = 0, gamma = 0, gammap = 0, gamrat = 1, crate = 1, acnrm = 0, saved_tq5 = 0;
  int q = 1, qprime = 1, L = 2, qwait = 2, qmax = 5;
  long long nst = 0, nfe = 0, nje = 0, nsetups = 0, nni = 0, netf = 0, ncfn = 0, nstlp = 0, nstlj = 0;

  GlobalRunner(GlobalBuffers& b, const Opts& oo, const P& p, cudaStream_t s, int nn, long long NN, const double* at,
               const double* fe, const double* ax)
      : B(b), o(oo), prm(p), st(s), n(nn), N(NN), M((long long)nn * NN), atol(at), fext(fe), aux(ax) {
    qmax = o.qmax;
  }

  unsigned gridc() const { return (unsigned)((N + 127) / 128); }
  unsigned gride() const { return (unsigned)((M + 255) / 256); }
  unsigned gridg() const { return (unsigned)((N * Model::G + 127) / 128); }
  size_t smemg() const { return sizeof(double) * (size_t)GMK<Model>::PG * GMK<Model>::GPB; }

  // ---- collective helpers (rank-ordered, deterministic) -------------------
  double allsum(double local) {
    if (!B.comm) return local;   // with a communicator the exchange always runs (nranks = 1 included)
    cudaMemcpyAsync(B.sum, &local, sizeof(double), cudaMemcpyHostToDevice, st);
    ncclAllGather(B.sum, B.gath, 1, ncclDouble, B.comm, st);
    std::vector<double> h(B.nranks);
    cudaMemcpyAsync(h.data(), B.gath, sizeof(double) * B.nranks, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double acc = 0.0;
    for (int r = 0; r < B.nranks; ++r) acc = acc + h[r];
    return acc;
  }
  int allor(int local) {
    if (!B.comm) return local;   // with a communicator the exchange always runs (nranks = 1 included)
    cudaMemcpyAsync(B.flag, &local, sizeof(int), cudaMemcpyHostToDevice, st);
    ncclAllGather(B.flag, B.igath, 1, ncclInt, B.comm, st);
    std::vector<int> h(B.nranks);
    cudaMemcpyAsync(h.data(), B.igath, sizeof(int) * B.nranks, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    int r = 0;
    for (int i = 0; i < B.nranks; ++i) r |= h[i];
    return r;
  }
  double allmax(double local) {
    if (!B.comm) return local;   // with a communicator the exchange always runs (nranks = 1 included)
    cudaMemcpyAsync(B.sum, &local, sizeof(double), cudaMemcpyHostToDevice, st);
    ncclAllGather(B.sum, B.gath, 1, ncclDouble, B.comm, st);
    std::vector<double> h(B.nranks);
    cudaMemcpyAsync(h.data(), B.gath, sizeof(double) * B.nranks, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double m = 0.0;
    for (int r = 0; r < B.nranks; ++r) m = fmax(m, h[r]);
    return m;
  }

  // WRMS over the whole batch (Eq. 3 with N = n * N_total, R14; order R15)
  double wrms(const double* x) {
    ++launches; gk_cellsum<<<gridc(), 128, 0, st>>>(x, B.v.ewt, B.s, n, N);
    const long long nb = (N + GM_BLK - 1) / GM_BLK;
    ++launches; gk_blocksum<<<(unsigned)((nb + 127) / 128), 128, 0, st>>>(B.s, B.P, N);
    ++launches; gk_finalsum<<<1, GK_FINAL_THREADS, 0, st>>>(B.P, nb, B.sum);
    double S = 0.0;
    cudaMemcpyAsync(&S, B.sum, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    S = allsum(S);
    return sqrt(S / ((double)n * (double)B.ncells_total));
  }

  int rhs(double t, const double* yin, double* fout) {
    cudaMemsetAsync(B.flag, 0, sizeof(int), st);
    if constexpr (TPC) {
      ++launches; gt_rhs<TM><<<gridc(), 128, 0, st>>>(N, yin, fext, aux, fout, B.flag);
    } else if constexpr (LANES) {
      ++launches; gl_rhs<Model><<<gridg(), 128, sizeof(double) * GLK<Model>::PG_RHS * GLK<Model>::GPB, st>>>(
          N, yin, fext, aux, fout, B.flag);
    } else {
      ++launches; gk_rhs<Model><<<gridg(), 128, smemg(), st>>>(prm, N, t, yin, fext, aux, fout, B.flag);
    }
    nfe++;
    int fl = 0;
    cudaMemcpyAsync(&fl, B.flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return allor(fl);
  }

  void ewt_from(const double* y) { ++launches; gk_ewt<<<gride(), 256, 0, st>>>(B.v.ewt, y, atol, o.rtol, n, N); }
  void rescale() {
    ++launches; gk_rescale<<<gridc(), 128, 0, st>>>(B.v, n, N, q, eta);
    h = hscale * eta;
    hscale = h;
  }
  void predict() {
    tn = tn + h;
    if ((tn - o.tf) * h > 0.0) tn = o.tf;
    ++launches; gk_predict<<<gridc(), 128, 0, st>>>(B.v, n, N, q);
  }
  void restore() {
    tn = saved_t;
    ++launches; gk_restore<<<gridc(), 128, 0, st>>>(B.v, n, N, q);
  }

  void set_bdf() {
    double xi_inv = 1.0, xistar_inv = 1.0, alpha0 = -1.0, alpha0_hat = -1.0, hsum = h;
    l[0] = l[1] = 1.0;
    for (int i = 2; i <= QMAX; ++i) l[i] = 0.0;
    if (q > 1) {
      for (int j = 2; j < q; ++j) {
        hsum = hsum + tau[j - 1];
        xi_inv = h / hsum;
        alpha0 = alpha0 - 1.0 / j;
        for (int i = j; i >= 1; --i) l[i] = l[i] + l[i - 1] * xi_inv;
      }
      alpha0 = alpha0 - 1.0 / q;
      xistar_inv = -l[1] - alpha0;
      hsum = hsum + tau[q - 1];
      xi_inv = h / hsum;
      alpha0_hat = -l[1] - xi_inv;
      for (int i = q; i >= 1; --i) l[i] = l[i] + l[i - 1] * xistar_inv;
    }
    const double A1 = 1.0 - alpha0_hat + alpha0;
    const double A2 = 1.0 + q * A1;
    tq[2] = fabs(A1 / (alpha0 * A2));
    tq[5] = fabs(A2 * xistar_inv / (l[q] * xi_inv));
    if (qwait == 1) {
      if (q > 1) {
        const double C = xistar_inv / l[q];
        const double A3 = alpha0 + 1.0 / q;
        const double A4 = alpha0_hat + xi_inv;
        const double Cpinv = (1.0 - A4 + A3) / A3;
        tq[1] = fabs(C * Cpinv);
      } else {
        tq[1] = 1.0;
      }
      hsum = hsum + tau[q];
      xi_inv = h / hsum;
      const double A5 = alpha0 - 1.0 / (q + 1);
      const double A6 = alpha0_hat - xi_inv;
      const double Cppinv = (1.0 - A6 + A5) / A2;
      tq[3] = fabs(Cppinv / (xi_inv * (q + 2) * A5));
    }
    tq[4] = NLSCOEF / tq[2];
  }

  void adjust_order(int dq) {
    if (q == 2 && dq != 1) return;
    GCoef lc{};
    if (dq == 1) {
      double alpha1 = 1.0, prod = 1.0, xiold = 1.0, alpha0 = -1.0, hsum = hscale;
      lc.c[2] = 1.0;
      if (q > 1) {
        for (int j = 1; j < q; ++j) {
          hsum = hsum + tau[j + 1];
          const double xi = hsum / hscale;
          prod = prod * xi;
          alpha0 = alpha0 - 1.0 / (j + 1);
          alpha1 = alpha1 + 1.0 / xi;
          for (int i = j + 2; i >= 2; --i) lc.c[i] = lc.c[i] * xiold + lc.c[i - 1];
          xiold = xi;
        }
      }
      const double A1 = (-alpha0 - alpha1) / prod;
      ++launches; gk_increase<<<gridc(), 128, 0, st>>>(B.v, n, N, q, qmax, A1, lc);
    } else {
      lc.c[2] = 1.0;
      double hsum = 0.0;
      for (int j = 1; j <= q - 2; ++j) {
        hsum = hsum + tau[j];
        const double xi = hsum / hscale;
        for (int i = j + 2; i >= 2; --i) lc.c[i] = lc.c[i] * xi + lc.c[i - 1];
      }
      ++launches; gk_decrease<<<gridc(), 128, 0, st>>>(B.v, n, N, q, lc);
    }
  }

  void set_eta() {
    if (eta < THRESH) {
      eta = 1.0;
      hprime = h;
    } else {
      eta = fmin(eta, etamax);
      if (o.hmax > 0.0) eta = eta / fmax(1.0, fabs(h) * eta / o.hmax);
      hprime = h * eta;
    }
  }

  // residual at ycor = acor: yq = zn0 + acor; f = R(tn, yq); del = -gamma f + (rl1 zn1 + acor)
  int residual() {
    ++launches; gk_axpby<<<gride(), 256, 0, st>>>(B.v.yq, 1.0, B.v.zn[0], 1.0, B.v.acor, M);
    const int r = rhs(tn, B.v.yq, B.v.f);
    if (r) return r;
    ++launches; gk_residual<<<gride(), 256, 0, st>>>(B.v, M, gamma, rl1);
    return 0;
  }

  int lsetup(int convfail, int& jcur) {
    const double dgamma = fabs(gamma / gammap - 1.0);
    const bool jbad = (nst == 0) || (nst >= nstlj + MSBJ) || (convfail == CF_BAD_J && dgamma < DGMAX_JBAD) ||
                      (convfail == CF_OTHER);
    if (jbad) {
      nje++;
      nstlj = nst;
      jcur = 1;
    } else {
      jcur = 0;
    }
    cudaMemsetAsync(B.flag, 0, sizeof(int), st);
    if constexpr (TPC && !LANES) {
      ++launches; gt_setup<TM><<<gridc(), 128, 0, st>>>(N, jbad ? 1 : 0, gamma, B.v.yq, aux, B.J, B.LU, B.perm,
                                                         B.invd, B.flag);
    } else if constexpr (LANES) {
      if (jbad) {   // J into HBM, then the register-row LU
        if (gl_jac2()) {   // the generated two-pass Jacobian of the SPLIT path (5 launches per 65536-cell chunk)
          const cudaError_t je = split_jac_diag(BDFB_MODEL_MECH_GRI53, N, B.v.yq, aux, B.J, B.flag, st);
          if (je != cudaSuccess) {   // e.g. no scratch: reported, and the setup fails (recoverably)
            fprintf(stderr, "bdfb: global-norm Jacobian: %s\n", cudaGetErrorString(je));
            cudaMemsetAsync(B.flag, 1, 1, st);
          }
          launches += 5 * (int)((N + 65535) / 65536);
        } else {           // BDFB_GLOBAL_JAC2=0: the table-driven lanes model
          ++launches; gl_setup<Model><<<gridg(), 128, sizeof(double) * GLK<Model>::PG_SET * GLK<Model>::GPB, st>>>(
              N, 1, gamma, B.v.yq, aux, B.J, B.LU, B.perm, B.invd, B.flag, 1);
        }
      }
      ++launches; gl_lu<Model::N><<<(unsigned)((N + GLU<Model::N>::CPB - 1) / GLU<Model::N>::CPB), GLU<Model::N>::T,
                                    gl_lu_smem<Model::N>(), st>>>(N, gamma, B.J, B.LU, B.perm, B.invd, B.flag);
    } else {
      ++launches; gk_setup<Model><<<gridg(), 128, smemg(), st>>>(prm, N, jbad ? 1 : 0, gamma, B.v.yq, aux, B.J, B.LU,
                                                                  B.pos, B.perm, B.invd, B.flag);
    }
    int fl = 0;
    cudaMemcpyAsync(&fl, B.flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fl = allor(fl);
    nsetups++;
    gamrat = 1.0;
    gammap = gamma;
    crate = 1.0;
    nstlp = nst;
    return fl ? 1 : 0;
  }

  int newton(int nflag) {
    int convfail = (nflag == NF_FIRST || nflag == NF_PREV_ERR) ? CF_NONE : CF_OTHER;
    int setup = (nflag == NF_PREV_CONV) || (nflag == NF_PREV_ERR) || (nst == 0) || (nst >= nstlp + MSBP) ||
                (fabs(gamrat - 1.0) > DGMAX);
    const double tol = tq[4];
    int jcur = 0;
    cudaMemsetAsync(B.v.acor, 0, sizeof(double) * M, st);
    for (;;) {
      int rv = residual();
      if (rv > 0) return 1;   // a failed first residual is not retried (reading R5)
      if (rv == 0 && setup) {
        rv = lsetup(convfail, jcur);
        setup = 0;
      }
      if (rv == 0) {
        double dprev = 0.0;
        int m = 0;
        for (;;) {
          nni++;
          const double sc2 = (gamrat != 1.0) ? 2.0 / (1.0 + gamrat) : 1.0;
          if constexpr (TPC && !LANES) {
            ++launches; gt_solve<TM><<<gridc(), 128, 0, st>>>(N, sc2, B.LU, B.perm, B.invd, B.v.del, B.v.acor,
                                                               B.v.tmp);
          } else if constexpr (LANES) {
            ++launches; gl_solve<Model::N><<<gridc(), 128, 0, st>>>(N, sc2, B.LU, B.perm, B.invd, B.v.del, B.v.acor,
                                                                    B.v.tmp);
          } else {
            ++launches; gk_solve<Model><<<gridg(), 128, smemg(), st>>>(N, sc2, B.LU, B.pos, B.perm, B.invd, B.v.del,
                                                                        B.v.acor, B.v.tmp);
          }
          const double del = wrms(B.v.tmp);
          if (m > 0) crate = fmax(CRDOWN * crate, del / dprev);
          const double dcon = del * fmin(1.0, crate) / tol;
          if (dcon <= 1.0) {
            acnrm = (m == 0) ? del : wrms(B.v.acor);
            return 0;
          }
          if (m >= 1 && del > RDIV * dprev) { rv = 1; break; }
          dprev = del;
          m++;
          if (m >= MAXCOR) { rv = 1; break; }
          rv = residual();
          if (rv) break;
        }
      }
      if (rv > 0 && !jcur) {
        setup = 1;
        convfail = CF_BAD_J;
        cudaMemsetAsync(B.v.acor, 0, sizeof(double) * M, st);
        continue;
      }
      return 1;
    }
  }

  void prepare_next(double dsm) {
    if (etamax == 1.0) {
      qwait = qwait > 2 ? qwait : 2;
      qprime = q;
      hprime = h;
      eta = 1.0;
      return;
    }
    const double etaq = 1.0 / (root_host(BIAS2 * dsm, L) + ADDON);
    if (qwait != 0) {
      eta = etaq;
      qprime = q;
      set_eta();
      return;
    }
    qwait = 2;
    double etaqm1 = 0.0, etaqp1 = 0.0;
    if (q > 1) {
      const double ddn = wrms(B.v.zn[q]) * tq[1];
      etaqm1 = 1.0 / (root_host(BIAS1 * ddn, q) + ADDON);
    }
    if (q != qmax && saved_tq5 != 0.0) {
      const double hr = h / tau[2];
      double pw = 1.0;
      for (int k = 0; k < L; ++k) pw = pw * hr;
      const double cquot = (tq[5] / saved_tq5) * pw;
      ++launches; gk_axpby<<<gride(), 256, 0, st>>>(B.v.tmp, -cquot, B.v.zn[qmax], 1.0, B.v.acor, M);
      const double dup = wrms(B.v.tmp) * tq[3];
      etaqp1 = 1.0 / (root_host(BIAS3 * dup, L + 1) + ADDON);
    }
    const double etam = fmax(etaqm1, fmax(etaq, etaqp1));
    if (etam < THRESH) {
      eta = 1.0;
      qprime = q;
    } else if (etam == etaq) {
      eta = etaq;
      qprime = q;
    } else if (etam == etaqm1) {
      eta = etaqm1;
      qprime = q - 1;
    } else {
      eta = etaqp1;
      qprime = q + 1;
      ++launches; gk_axpby<<<gride(), 256, 0, st>>>(B.v.zn[qmax], 1.0, B.v.acor, 0.0, nullptr, M);
    }
    set_eta();
  }

  int hin(double& h0) {
    const double tdist = o.tf - o.t0;
    const double tround = UROUND * fmax(fabs(o.t0), fabs(o.tf));
    const double hlb = 100.0 * tround;
    cudaMemsetAsync(B.ubuf, 0, sizeof(unsigned long long), st);
    ++launches; gk_hubinv<<<gride(), 256, 0, st>>>(B.v, M, B.ubuf);
    unsigned long long bits = 0;
    cudaMemcpyAsync(&bits, B.ubuf, sizeof(bits), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double hub_inv;
    memcpy(&hub_inv, &bits, sizeof(double));
    hub_inv = allmax(hub_inv);
    double hub = HUB_FACTOR * tdist;
    if (hub * hub_inv > 1.0) hub = 1.0 / hub_inv;
    double hg = sqrt(hlb * hub);
    if (hub < hlb) { h0 = hg; return 0; }
    double hs = hg, hnew = hg;
    for (int count1 = 1; count1 <= HIN_ITERS; ++count1) {
      int ok = 0;
      double ydd = 0.0;
      for (int count2 = 1; count2 <= HIN_ITERS; ++count2) {
        ++launches; gk_axpby<<<gride(), 256, 0, st>>>(B.v.yq, hg, B.v.zn[1], 1.0, B.v.zn[0], M);
        const int r = rhs(o.t0 + hg, B.v.yq, B.v.f);
        if (r == 0) {
          const double ih = 1.0 / hg;
          // tmp = (f - f0) * (1/hg)
          ++launches; gk_axpby<<<gride(), 256, 0, st>>>(B.v.tmp, 1.0, B.v.f, -1.0, B.v.zn[1], M);
          ++launches; gk_axpby<<<gride(), 256, 0, st>>>(B.v.tmp, ih, B.v.tmp, 0.0, nullptr, M);
          ydd = wrms(B.v.tmp);
          ok = 1;
          break;
        }
        hg = hg * 0.2;
      }
      if (!ok) {
        if (count1 <= 2) return -1;
        hnew = hs;
        break;
      }
      hs = hg;
      hnew = (ydd * hub * hub > 2.0) ? sqrt(2.0 / ydd) : sqrt(hg * hub);
      if (count1 == HIN_ITERS) break;
      const double hrat = hnew / hg;
      if (hrat > 0.5 && hrat < 2.0) break;
      if (count1 > 1 && hrat > 2.0) { hnew = hg; break; }
      hg = hnew;
    }
    double hh = H_BIAS * hnew;
    if (hh < hlb) hh = hlb;
    if (hh > hub) hh = hub;
    h0 = hh;
    return 0;
  }

  static double root_host(double x, int Lr) {   // reading R25, host copy of root_l's sequence
    static const double C[8][7] = {
        {0}, {1.0},
        {0x1.0p+0, 0x1.6a09e667f3bcdp+0},
        {0x1.0p+0, 0x1.428a2f98d728bp+0, 0x1.965fea53d6e3dp+0},
        {0x1.0p+0, 0x1.306fe0a31b715p+0, 0x1.6a09e667f3bcdp+0, 0x1.ae89f995ad3adp+0},
        {0x1.0p+0, 0x1.2611186bae675p+0, 0x1.51cb453b9536cp+0, 0x1.8406003b2ae5cp+0, 0x1.bdb8cdadbe120p+0},
        {0x1.0p+0, 0x1.1f59ac3c7d6c0p+0, 0x1.428a2f98d728bp+0, 0x1.6a09e667f3bcdp+0, 0x1.965fea53d6e3dp+0,
         0x1.c823e074ec129p+0},
        {0x1.0p+0, 0x1.1aa59c4115e7dp+0, 0x1.381147622f886p+0, 0x1.588cea3f093bep+0, 0x1.7c6a1f29e2ce6p+0,
         0x1.a402feeb9c533p+0, 0x1.cfbb031a741a5p+0}};
    static const double CL[8] = {0, 0, 0x1.2bec333018867p-2, 0x1.a68056b0a470ep-3, 0x1.45d819a94b14bp-3,
                                 0x1.091cc94907b7fp-3, 0x1.bee0fc589f6b6p-4, 0x1.8227e72c5f2dbp-4};
    if (!(x > 0.0) || isinf(x)) return x > 0.0 ? x : 0.0;
    if (Lr == 1) return x;
    int e;
    const double y = 2.0 * frexp(x, &e);
    e = e - 1;
    const int k = (e >= 0) ? e / Lr : -((-e + Lr - 1) / Lr);
    const int r = e - Lr * k;
    const double invL = 1.0 / Lr;
    double s = 1.0 - (y - 1.0) * CL[Lr];
    for (int it = 0; it < 4; ++it) {
      double p = s;
      for (int j = 0; j < Lr - 1; ++j) p = p * s;
      s = s * (1.0 + (1.0 - y * p) * invL);
    }
    double t = y;
    for (int j = 0; j < Lr - 1; ++j) t = t * s;
    return ldexp(t * C[Lr][r], k);
  }

  // one accepted step (cvStep); returns ST_OK or a failure status
  int step() {
    saved_t = tn;
    int ncf = 0, nef = 0, nflag = NF_FIRST;
    if (nst > 0 && hprime != h) {
      if (qprime != q) {
        adjust_order(qprime - q);
        q = qprime;
        L = q + 1;
        qwait = L;
      }
      rescale();
    }
    double dsm;
    for (;;) {
      predict();
      set_bdf();
      rl1 = 1.0 / l[1];
      gamma = h * rl1;
      if (nst == 0) gammap = gamma;
      gamrat = (nst > 0) ? gamma / gammap : 1.0;
      const int r = newton(nflag);
      if (r) {
        ncfn++;
        restore();
        ncf++;
        etamax = 1.0;
        if (fabs(h) <= o.hmin * (1.0 + UROUND) || ncf == MXNCF) return ST_CONV_FAILURE;
        eta = fmax(ETACF, o.hmin / fabs(h));
        nflag = NF_PREV_CONV;
        rescale();
        continue;
      }
      dsm = acnrm * tq[2];
      if (dsm <= 1.0) break;
      nef++;
      netf++;
      nflag = NF_PREV_ERR;
      restore();
      if (fabs(h) <= o.hmin * (1.0 + UROUND) || nef == MXNEF) return ST_ERR_FAILURE;
      etamax = 1.0;
      if (nef <= MXNEF1) {
        eta = 1.0 / (root_host(BIAS2 * dsm, L) + ADDON);
        eta = fmax(ETAMIN, fmax(eta, o.hmin / fabs(h)));
        if (nef >= SMALL_NEF) eta = fmin(eta, ETAMXF);
        rescale();
        continue;
      }
      if (q > 1) {
        eta = fmax(ETAMIN, o.hmin / fabs(h));
        adjust_order(-1);
        L = q;
        q = q - 1;
        qwait = L;
        rescale();
        continue;
      }
      eta = fmax(ETAMIN, o.hmin / fabs(h));
      h = h * eta;
      hprime = h;
      hscale = h;
      qwait = LONG_WAIT;
      if (rhs(tn, B.v.zn[0], B.v.f)) return ST_RHS_FAIL;
      ++launches; gk_axpby<<<gride(), 256, 0, st>>>(B.v.zn[1], h, B.v.f, 0.0, nullptr, M);
    }
    nst++;
    for (int i = q; i >= 2; --i) tau[i] = tau[i - 1];
    if (q == 1 && nst > 1) tau[2] = tau[1];
    tau[1] = h;
    qwait--;
    const int save = (qwait == 1 && q != qmax);
    GCoef lco{};
    for (int j = 0; j <= QMAX; ++j) lco.c[j] = l[j];
    ++launches; gk_complete<<<gridc(), 128, 0, st>>>(B.v, n, N, q, lco, save, qmax);
    if (save) saved_tq5 = tq[5];
    prepare_next(dsm);
    etamax = ETAMX2;
    return ST_OK;
  }

  GlobalResult run(double* y) {
    GlobalResult res{};
    res.status = ST_OK;
    res.tn = o.t0;
    // non-finite input anywhere -> the batch is not integrated
    cudaMemsetAsync(B.flag, 0, sizeof(int), st);
    ++launches; gk_finite<<<gride(), 256, 0, st>>>(y, M, B.flag);
    if (fext) { ++launches; gk_finite<<<gride(), 256, 0, st>>>(fext, M, B.flag); }
    int fl = 0;
    cudaMemcpyAsync(&fl, B.flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (allor(fl)) { res.status = ST_NONFINITE; return res; }
    cudaMemcpyAsync(B.v.zn[0], y, sizeof(double) * M, cudaMemcpyDeviceToDevice, st);
    ewt_from(B.v.zn[0]);
    tn = o.t0;
    int status = ST_OK;
    double h0 = o.h0;
    if (rhs(o.t0, B.v.zn[0], B.v.zn[1])) {
      status = ST_RHS_FAIL;
    } else if (h0 == 0.0 && hin(h0)) {
      status = ST_RHS_FAIL;
    }
    if (status == ST_OK) {
      if (h0 > o.tf - o.t0) h0 = o.tf - o.t0;
      if (o.hmax > 0.0 && h0 > o.hmax) h0 = o.hmax;
      ++launches; gk_axpby<<<gride(), 256, 0, st>>>(B.v.zn[1], h0, B.v.zn[1], 0.0, nullptr, M);
      h = hscale = hprime = h0;
      q = qprime = 1;
      L = 2;
      qwait = 2;
      etamax = ETAMX1;
      crate = 1.0;
      eta = 1.0;
      for (;;) {
        if (nst > 0) ewt_from(B.v.zn[0]);
        if ((tn + hprime - o.tf) * h > 0.0) {
          hprime = o.tf - tn;
          eta = hprime / h;
        }
        if (nst >= o.mxstep) { status = ST_TOO_MUCH_WORK; break; }
        const int r = step();
        if (r != ST_OK) { status = r; break; }
        if (fabs(tn - o.tf) <= 100.0 * UROUND * (fabs(tn) + fabs(h))) {
          tn = o.tf;
          break;
        }
      }
      cudaMemcpyAsync(y, B.v.zn[0], sizeof(double) * M, cudaMemcpyDeviceToDevice, st);
    }
    cudaStreamSynchronize(st);
    res.status = status;
    res.nst = nst; res.nfe = nfe; res.nje = nje; res.nsetups = nsetups; res.nni = nni; res.netf = netf;
    res.ncfn = ncfn; res.q = q; res.h = h; res.tn = tn; res.launches = launches;
    return res;
  }
};

}  // namespace bdfb
