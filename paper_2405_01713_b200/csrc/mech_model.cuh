// mech_model.cuh -- constant-volume, constant-internal-energy reactor RHS and
// analytic Jacobian for a generated mechanism (T = gen/mech_<name>.cuh
// Traits), one cell per group of G lanes.
//
// Physics (the paper's 0-D reactor "assumed constant
// internal energy", split form dU/dt = F + R):
//   C_k = rho Y_k / W_k;  k_f = exp(ln A + beta ln T - Ea/(R_c T));
//   [M] = sum_k alpha_k C_k;  Lindemann / Troe falloff;
//   1/K_c = prod_reac e^{-g/RT} / prod_prod e^{-g/RT} * (R T / p_atm)^{dnu};
//   q = k_f (prod_reac C - prod_prod C / K_c)  (times [M] for third body);
//   wdot_k = sum_r nu_rk q_r;  dY_k/dt = W_k wdot_k / rho;
//   dT/dt = -sum_k u_k wdot_k / (rho cv),  u_k = (h_k/RT - 1) R T.
// The analytic Jacobian ("generated offline, mechanism-specific") is
// the exact derivative of that RHS: d/dC through the mass-action products,
// [M] and the falloff blending, d/dT through k_f, K_c, Troe F_cent, u and cv.
//
// GPU organisation per group: (1) lanes = species: concentrations, NASA-7
// thermo, e^{-g/RT} (one exp per species instead of one per reaction);
// (2) lanes = reactions (ceil(NR/G) rounds): rates of progress to shared
// memory; (3) lanes = species: padded-ELL gather of wdot (branch-free), the
// T row by two butterfly reductions.  The Jacobian (cold path, outlined) adds
// per-reaction partial derivatives, written into the LU area that the matrix
// setup overwrites right after, and a row-per-lane assembly in shared memory.
#pragma once
#include "grp.cuh"
#include "lu.cuh"

namespace bdfb {

template <class T>
struct ModelMech {
  static constexpr int K = T::K, N = T::N, G = T::G, NR = T::NR, NTB = T::NTB, ELL = T::ELL;
  static constexpr bool DIAG = false;
#ifndef BDFB_MECH_BLOCK
#define BDFB_MECH_BLOCK 128
#endif
#ifndef BDFB_MECH_MINB
#define BDFB_MECH_MINB 3
#endif
  static constexpr int BLOCK = BDFB_MECH_BLOCK;
  static constexpr int MINB = BDFB_MECH_MINB;           // target resident blocks per SM
  static constexpr int GPW = 32 / G;                    // groups per warp
  static constexpr int ROUNDS = (NR + G - 1) / G;
  // shared scratch per group (doubles); q[NR] is a zero slot for ELL padding
  static constexpr int O_Y = 0, O_C = N, O_G = O_C + K, O_H = O_G + K, O_CP = O_H + K, O_EG = O_CP + K,
                       O_Q = O_EG + K, SG = O_Q + NR + 1;
  // Jacobian-only scratch per group (lives in the LU area)
  static constexpr int J_DR = 0, J_DP = 3 * NR, J_DM = 6 * NR, J_DT = 7 * NR, JG = 8 * NR;
  static constexpr int SCRATCH = GPW * SG;
  static constexpr int JSCRATCH = GPW * JG;
  static constexpr double RU = 8.31446261815324e7, PATM = 1013250.0, LN10 = 2.302585092994045684;
  struct Params { double unused; };

  // scratch pointers passed to rhs()/jac() are the GROUP's own (SG doubles;
  // Jacobian scratch JG doubles); matrix rows: row[j * stride] is (lane, j).

  // phase 1: broadcast y, species thermo.  Returns 1 if T is not positive.
  __device__ static int species(const Grp<G>& g, double y, double rho, double* sc, double& Tt, double& lnT,
                                double& invT) {
    if (g.lane < N) sc[O_Y + g.lane] = y;
    if (g.lane == 0) sc[O_Q + NR] = 0.0;
    g.sync();
    Tt = sc[O_Y + K];
    if (!(Tt > 0.0)) return 1;
    lnT = log(Tt);
    invT = 1.0 / Tt;
    const int k = g.lane;
    if (k < K) {
      const double* a = (Tt < T::Tmid()[k]) ? T::nasa_lo() : T::nasa_hi();
      const double a0 = a[k], a1 = a[K + k], a2 = a[2 * K + k], a3 = a[3 * K + k], a4 = a[4 * K + k],
                   a5 = a[5 * K + k], a6 = a[6 * K + k];
      const double cp = fma(Tt, fma(Tt, fma(Tt, fma(Tt, a4, a3), a2), a1), a0);
      const double h = fma(Tt, fma(Tt, fma(Tt, fma(Tt, a4 * 0.2, a3 * 0.25), a2 * (1.0 / 3.0)), a1 * 0.5), a0) +
                       a5 * invT;
      const double s = fma(a0, lnT, fma(Tt, fma(Tt, fma(Tt, fma(Tt, a4 * 0.25, a3 * (1.0 / 3.0)), a2 * 0.5), a1), a6));
      const double gk = h - s;
      sc[O_C + k] = rho * sc[O_Y + k] * T::invW()[k];
      sc[O_G + k] = gk;
      sc[O_H + k] = h;
      sc[O_CP + k] = cp;
      sc[O_EG + k] = exp(-gk);
    }
    g.sync();
    return 0;
  }

  // phase 2: rates of progress (and partial derivatives into js if DERIV)
  template <bool DERIV>
  __device__ static void reactions(const Grp<G>& g, double* sc, double* js, double Tt, double lnT, double invT) {
    const double cRT = RU * Tt / PATM, icRT = PATM / (RU * Tt);
#pragma unroll 1
    for (int rr = 0; rr < ROUNDS; ++rr) {
      const int r = rr * G + g.lane;
      if (r < NR) {
        const int ty = T::rtype()[r];
        const int i0 = T::reac0()[r], i1 = T::reac1()[r], i2 = T::reac2()[r];
        const int j0 = T::prod0()[r], j1 = T::prod1()[r], j2 = T::prod2()[r];
        const double c0 = sc[O_C + i0];
        const double c1 = i1 >= 0 ? sc[O_C + i1] : 1.0;
        const double c2 = i2 >= 0 ? sc[O_C + i2] : 1.0;
        const double p0 = sc[O_C + j0];
        const double p1 = j1 >= 0 ? sc[O_C + j1] : 1.0;
        const double p2 = j2 >= 0 ? sc[O_C + j2] : 1.0;
        const double Cf = c0 * c1 * c2;
        const double Cr = p0 * p1 * p2;
        double invKc = 0.0, dlnKc = 0.0;
        if (T::rev()[r]) {
          const double er = sc[O_EG + i0] * (i1 >= 0 ? sc[O_EG + i1] : 1.0) * (i2 >= 0 ? sc[O_EG + i2] : 1.0);
          const double ep = sc[O_EG + j0] * (j1 >= 0 ? sc[O_EG + j1] : 1.0) * (j2 >= 0 ? sc[O_EG + j2] : 1.0);
          const int dn = T::dnu()[r];
          const double cf = dn == 0 ? 1.0 : (dn == 1 ? cRT : (dn == -1 ? icRT : (dn > 0 ? cRT * cRT : icRT * icRT)));
          invKc = er / ep * cf;
          if (DERIV) {
            double hs = sc[O_H + j0] - sc[O_H + i0];
            if (j1 >= 0) hs += sc[O_H + j1];
            if (j2 >= 0) hs += sc[O_H + j2];
            if (i1 >= 0) hs -= sc[O_H + i1];
            if (i2 >= 0) hs -= sc[O_H + i2];
            dlnKc = (hs - dn) * invT;
          }
        }
        const double b = T::beta()[r], ea = T::EaR()[r];
        // constant-rate reactions (beta = Ea = 0) are grouped into whole rounds by the codegen
#ifdef BDFB_NO_KCONST
        const double kinf = exp(fma(b, lnT, T::lnA()[r]) - ea * invT);
#else
        const double kinf = T::kconst()[r] ? T::Aconst()[r] : exp(fma(b, lnT, T::lnA()[r]) - ea * invT);
#endif
        const double net = fma(-Cr, invKc, Cf);
        double k = kinf, M = 1.0, dkdT = 0.0, dkdM = 0.0;
        if (DERIV) dkdT = kinf * (b + ea * invT) * invT;
        if (ty >= 1) {
          const double* e = T::eff() + T::tbidx()[r] * K;
          double M0 = 0.0, M1 = 0.0;
#pragma unroll 4
          for (int j = 0; j + 1 < K; j += 2) {
            M0 = fma(e[j], sc[O_C + j], M0);
            M1 = fma(e[j + 1], sc[O_C + j + 1], M1);
          }
          if (K & 1) M0 = fma(e[K - 1], sc[O_C + K - 1], M0);
          M = M0 + M1;
          if (ty >= 2) {
            const double b0 = T::beta0()[r], ea0 = T::EaR0()[r];
            const double k0 = exp(fma(b0, lnT, T::lnA0()[r]) - ea0 * invT);
            const double Pr = k0 * M / kinf;
            const double Pr1 = 1.0 / (1.0 + Pr);
            double F = 1.0, dlFdlPr = 0.0, dFdT = 0.0;
            if (ty == 3) {
              const double a = T::troe_a()[r], iT3 = T::troe_iT3()[r], iT1 = T::troe_iT1()[r];
              const double e3 = exp(-Tt * iT3), e1 = exp(-Tt * iT1);
              double Fc = (1.0 - a) * e3 + a * e1;
              double dFc = 0.0;
              if (DERIV) dFc = -(1.0 - a) * iT3 * e3 - a * iT1 * e1;
              if (T::troe_has_t2()[r]) {
                const double T2 = T::troe_T2()[r];
                const double e2 = exp(-T2 * invT);
                Fc += e2;
                if (DERIV) dFc += T2 * invT * invT * e2;
              }
              const double lFc = log10(Fc);
              const double cc = -0.4 - 0.67 * lFc, nn = 0.75 - 1.27 * lFc;
              const double x = log10(Pr) + cc;
              const double den = 1.0 / (nn - 0.14 * x);
              const double f1 = x * den;
              const double q1 = 1.0 / (1.0 + f1 * f1);
              const double lF = lFc * q1;
              F = exp(lF * LN10);
              if (DERIV) {
                const double df1dx = nn * den * den;
                dlFdlPr = -lFc * 2.0 * f1 * df1dx * q1 * q1;
                const double df1dlFc = (-0.67 * (nn - 0.14 * x) - x * (-1.27 + 0.14 * 0.67)) * den * den;
                const double dlFdlFc = q1 - lFc * 2.0 * f1 * df1dlFc * q1 * q1;
                const double dlFcdT = dFc / (Fc * LN10);
                dFdT = F * LN10 * dlFdlFc * dlFcdT;
              }
            }
            const double gfac = Pr * Pr1 * F;
            k = kinf * gfac;
            if (DERIV) {
              // dg/dPr = F/(1+Pr)^2 + Pr/(1+Pr) dF/dPr,  dF/dPr = F dlF/dlPr / Pr
              const double dgdPr = F * Pr1 * Pr1 + Pr1 * F * dlFdlPr;
              const double dlnkinf = (b + ea * invT) * invT;
              const double dlnk0 = (b0 + ea0 * invT) * invT;
              dkdT = k * dlnkinf + kinf * dgdPr * Pr * (dlnk0 - dlnkinf) + kinf * Pr * Pr1 * dFdT;
              dkdM = k0 * dgdPr;
            }
            M = 1.0;
          }
        }
        const double q = M * k * net;
        sc[O_Q + r] = q;
        if (DERIV) {
          const double kf = M * k, kr = M * k * invKc;
          double* dr = js + J_DR;
          double* dp = js + J_DP;
          dr[r] = kf * c1 * c2;
          dr[NR + r] = i1 >= 0 ? kf * c0 * c2 : 0.0;
          dr[2 * NR + r] = i2 >= 0 ? kf * c0 * c1 : 0.0;
          dp[r] = -kr * p1 * p2;
          dp[NR + r] = j1 >= 0 ? -kr * p0 * p2 : 0.0;
          dp[2 * NR + r] = j2 >= 0 ? -kr * p0 * p1 : 0.0;
          js[J_DM + r] = ty == 1 ? k * net : (ty >= 2 ? dkdM * net : 0.0);
          js[J_DT + r] = M * (dkdT * net + k * Cr * invKc * dlnKc);
        }
      }
    }
    g.sync();
  }

  // wdot_k for this lane's species (k = lane < K): padded ELL, branch-free
  __device__ static double wdot(const Grp<G>& g, const double* sc) {
    const int k = g.lane < K ? g.lane : 0;
    double w0 = 0.0, w1 = 0.0;
#pragma unroll 4
    for (int m = 0; m + 1 < ELL; m += 2) {
      w0 = fma(T::ell_nu()[m * K + k], sc[O_Q + T::ell_r()[m * K + k]], w0);
      w1 = fma(T::ell_nu()[(m + 1) * K + k], sc[O_Q + T::ell_r()[(m + 1) * K + k]], w1);
    }
    if (ELL & 1) w0 = fma(T::ell_nu()[(ELL - 1) * K + k], sc[O_Q + T::ell_r()[(ELL - 1) * K + k]], w0);
    return g.lane < K ? w0 + w1 : 0.0;
  }

  __device__ static int rhs(const Grp<G>& g, const Params&, double, const double (&y)[1], double (&f)[1],
                            double rho, double* sc) {
    double Tt, lnT, invT;
    f[0] = 0.0;
    if (species(g, y[0], rho, sc, Tt, lnT, invT)) return 1;
    reactions<false>(g, sc, nullptr, Tt, lnT, invT);
    const int k = g.lane;
    const double w = wdot(g, sc);
    double cvp = 0.0, up = 0.0;
    if (k < K) {
      f[0] = T::W()[k] * w / rho;
      cvp = sc[O_Y + k] * (sc[O_CP + k] - 1.0) * RU * T::invW()[k];
      up = (sc[O_H + k] - 1.0) * RU * Tt * w;
    }
    const double cv = g.sum(cvp), su = g.sum(up);
    if (k == K) f[0] = -su / (rho * cv);
    g.sync();
    return 0;
  }

  // Analytic Jacobian: this lane's row at row[j * WS_] (j = 0..N-1); sc: the
  // group's SG scratch doubles; js: the group's JG Jacobian-scratch doubles
  // (inside the LU area, which the matrix setup overwrites right after).
  template <int WS_>
  __device__ static __noinline__ int jac(const Grp<G> g, double y, double rho, double* row, double* sc, double* js) {
    double Tt, lnT, invT;
    if (species(g, y, rho, sc, Tt, lnT, invT)) return 1;
    reactions<true>(g, sc, js, Tt, lnT, invT);
    const int k = g.lane;
    constexpr int WS = WS_;
    const double w = wdot(g, sc);
    if (k < N)
      for (int j = 0; j < N; ++j) row[j * WS] = 0.0;
    if (k < K) {
      const int len = T::ell_len()[k];
      double dT = 0.0;
      const double* dr = js + J_DR;
      const double* dp = js + J_DP;
      for (int m = 0; m < len; ++m) {
        const int r = T::ell_r()[m * K + k];
        const double nu = T::ell_nu()[m * K + k];
        int s;
        s = T::reac0()[r]; row[s * WS] = fma(nu, dr[r], row[s * WS]);
        s = T::reac1()[r]; if (s >= 0) row[s * WS] = fma(nu, dr[NR + r], row[s * WS]);
        s = T::reac2()[r]; if (s >= 0) row[s * WS] = fma(nu, dr[2 * NR + r], row[s * WS]);
        s = T::prod0()[r]; row[s * WS] = fma(nu, dp[r], row[s * WS]);
        s = T::prod1()[r]; if (s >= 0) row[s * WS] = fma(nu, dp[NR + r], row[s * WS]);
        s = T::prod2()[r]; if (s >= 0) row[s * WS] = fma(nu, dp[2 * NR + r], row[s * WS]);
        dT = fma(nu, js[J_DT + r], dT);
      }
      // third-body / falloff [M] dependence: dense in the collision partners
#pragma unroll 1
      for (int t = 0; t < NTB; ++t) {
        const double coef = T::nu_tb()[t * K + k] * js[J_DM + T::tb_rxn()[t]];
        if (coef != 0.0) {
          const double* e = T::eff() + t * K;
          for (int j = 0; j < K; ++j) row[j * WS] = fma(coef, e[j], row[j * WS]);
        }
      }
      // dY_k/dY_j = (W_k/W_j) sum nu dq/dC_j ;  dY_k/dT = (W_k/rho) sum nu dq/dT
      const double Wk = T::W()[k];
      for (int j = 0; j < K; ++j) row[j * WS] = row[j * WS] * (Wk * T::invW()[j]);
      row[K * WS] = Wk * dT / rho;
    }
    g.sync();
    // temperature row: f_T = -sum_k u_k wdot_k / (rho cv)
    double cvp = 0.0, up = 0.0, dcvp = 0.0, cvw = 0.0, uoW = 0.0;
    if (k < K) {
      const double Y = sc[O_Y + k];
      const double iW = T::invW()[k];
      const double u = (sc[O_H + k] - 1.0) * RU * Tt;
      cvp = Y * (sc[O_CP + k] - 1.0) * RU * iW;
      up = u * w;
      const double* a = (Tt < T::Tmid()[k]) ? T::nasa_lo() : T::nasa_hi();
      const double dcp = fma(Tt, fma(Tt, fma(Tt, 4.0 * a[4 * K + k], 3.0 * a[3 * K + k]), 2.0 * a[2 * K + k]),
                             a[K + k]);
      dcvp = Y * dcp * RU * iW;
      cvw = (sc[O_CP + k] - 1.0) * RU * w;
      uoW = u * iW;
    }
    const double cv = g.sum(cvp), su = g.sum(up), dcv = g.sum(dcvp), scw = g.sum(cvw);
    const double fT0 = -su / (rho * cv);
    const double icv = 1.0 / cv;
    for (int j = 0; j < N; ++j) {
      const double v = (k < K) ? uoW * row[j * WS] : 0.0;
      const double s = g.sum(v);
      if (k == K) {
        if (j < K) {
          const double cvj = (sc[O_CP + j] - 1.0) * RU * T::invW()[j];
          row[j * WS] = -s * icv - fT0 * cvj * icv;
        } else {
          row[j * WS] = -scw / (rho * cv) - s * icv - fT0 * dcv * icv;
        }
      }
    }
    g.sync();
    return 0;
  }
};

}  // namespace bdfb
