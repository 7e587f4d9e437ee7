// mech_lanes.cuh -- table-driven constant-volume reactor RHS and analytic
// Jacobian for ONE cell owned by a group of G lanes, any system size n:
// lane l owns components (species) i = l + G r, r < R = ceil(n / G)
// (the component distribution of reading R15, so the group's WRMS order is
// the oracle's order for G).  T = a generated gen/mech_<name>.cuh Traits.
//
// Physics: SURVEY.md §8(c).6 (the paper's 0-D reactor "assumed constant
// internal energy"; split form P:196-201), identical to
// mech_model.cuh (which holds one species per lane, n <= G):
//   C_k = rho Y_k / W_k;  k_f = exp(ln A + beta ln T - Ea/(R_c T));
//   [M] = sum_k alpha_k C_k;  Lindemann / Troe falloff;
//   1/K_c = prod_reac e^{-g/RT} / prod_prod e^{-g/RT} (R T / p_atm)^{dnu};
//   q = k_f (prod_reac C - prod_prod C / K_c) (times [M] for third body);
//   wdot_k = sum_r nu_rk q_r;  dY_k/dt = W_k wdot_k / rho;
//   dT/dt = -sum_k u_k wdot_k / (rho cv),  u_k = (h_k/RT - 1) R T.
// The analytic Jacobian ("generated offline, mechanism-specific") is
// the exact derivative of that RHS (chain rule through the mass-action
// products, [M], the falloff blending, k_f(T), K_c(T), F_cent(T), u and cv).
//
// Organisation per group (a warp holds 32/G groups; every phase is uniform
// code over table entries, so groups of one warp never diverge by mechanism
// structure): (1) lanes = species (R rounds): C, NASA-7 thermo, e^{-g/RT};
// (2) lanes = reactions (ceil(NR/G) rounds): rates of progress into shared
// scratch; (3) lanes = species: padded-ELL gather of wdot; the temperature
// row by two group butterflies.  Shared scratch per group: SG doubles (RHS),
// JG doubles (Jacobian partials, reusable after jac returns).
#pragma once
#include "fexp.cuh"
#include "grp.cuh"

namespace bdfb {

template <class T, int G_>
struct ModelMechR {
  static constexpr int K = T::K, N = T::N, G = G_, NR = T::NR, NTB = T::NTB, ELL = T::ELL;
  static constexpr int R = (N + G - 1) / G;            // components per lane
  static constexpr int ROUNDS = (NR + G - 1) / G;
  static constexpr int O_Y = 0, O_C = N, O_G = O_C + K, O_H = O_G + K, O_CP = O_H + K, O_EG = O_CP + K,
                       O_Q = O_EG + K, SG = O_Q + NR + 1;
  static constexpr int J_DR = 0, J_DP = 3 * NR, J_DM = 6 * NR, J_DT = 7 * NR, JG = 8 * NR;
  static constexpr double RU = 8.31446261815324e7, PATM = 1013250.0, LN10 = 2.302585092994045684;
  static constexpr bool LANES = true;      // global_host.cuh: drive with the global_lanes.cuh kernels
  struct Params { double unused; };

  // phase 1: y to scratch, species thermo.  Returns 1 if T is not positive (recoverable RHS failure).
  __device__ static int species(const Grp<G>& g, const double (&y)[R], double rho, double* sc, double& Tt,
                                double& lnT, double& invT) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = g.lane + G * r;
      if (i < N) sc[O_Y + i] = y[r];
    }
    if (g.lane == 0) sc[O_Q + NR] = 0.0;
    g.sync();
    Tt = sc[O_Y + K];
    if (!(Tt > 0.0)) return 1;
    lnT = log(Tt);
    invT = 1.0 / Tt;
#pragma unroll
    for (int r = 0; r < (K + G - 1) / G; ++r) {
      const int k = g.lane + G * r;
      if (k < K) {
        const double* a = (Tt < T::Tmid()[k]) ? T::nasa_lo() : T::nasa_hi();
        const double a0 = a[k], a1 = a[K + k], a2 = a[2 * K + k], a3 = a[3 * K + k], a4 = a[4 * K + k],
                     a5 = a[5 * K + k], a6 = a[6 * K + k];
        const double cp = fma(Tt, fma(Tt, fma(Tt, fma(Tt, a4, a3), a2), a1), a0);
        const double h = fma(Tt, fma(Tt, fma(Tt, fma(Tt, a4 * 0.2, a3 * 0.25), a2 * (1.0 / 3.0)), a1 * 0.5), a0) +
                         a5 * invT;
        const double s =
            fma(a0, lnT, fma(Tt, fma(Tt, fma(Tt, fma(Tt, a4 * 0.25, a3 * (1.0 / 3.0)), a2 * 0.5), a1), a6));
        const double gk = h - s;
        sc[O_C + k] = rho * sc[O_Y + k] * T::invW()[k];
        sc[O_G + k] = gk;
        sc[O_H + k] = h;
        sc[O_CP + k] = cp;
        sc[O_EG + k] = fexp(-gk);
      }
    }
    g.sync();
    return 0;
  }

  // phase 2: rates of progress q_r (and, with DERIV, their partial derivatives into js)
  template <bool DERIV>
  __device__ static void reactions(const Grp<G>& g, double* sc, double* js, double Tt, double lnT, double invT) {
    const double cRT = RU * Tt / PATM, icRT = PATM / (RU * Tt);
#pragma unroll 1
    for (int rr = 0; rr < ROUNDS; ++rr) {
      const int r = rr * G + g.lane;
      if (r >= NR) continue;
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
      const double kinf = T::kconst()[r] ? T::Aconst()[r] : fexp(fma(b, lnT, T::lnA()[r]) - ea * invT);
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
          const double k0 = fexp(fma(b0, lnT, T::lnA0()[r]) - ea0 * invT);
          const double Pr = k0 * M / kinf;
          const double Pr1 = 1.0 / (1.0 + Pr);
          double F = 1.0, dlFdlPr = 0.0, dFdT = 0.0;
          if (ty == 3) {
            const double a = T::troe_a()[r], iT3 = T::troe_iT3()[r], iT1 = T::troe_iT1()[r];
            const double e3 = fexp(-Tt * iT3), e1 = fexp(-Tt * iT1);
            double Fc = (1.0 - a) * e3 + a * e1;
            double dFc = 0.0;
            if (DERIV) dFc = -(1.0 - a) * iT3 * e3 - a * iT1 * e1;
            if (T::troe_has_t2()[r]) {
              const double T2 = T::troe_T2()[r];
              const double e2 = fexp(-T2 * invT);
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
            F = fexp(lF * LN10);
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
            const double dgdPr = F * Pr1 * Pr1 + Pr1 * F * dlFdlPr;
            const double dlnkinf = (b + ea * invT) * invT;
            const double dlnk0 = (b0 + ea0 * invT) * invT;
            dkdT = k * dlnkinf + kinf * dgdPr * Pr * (dlnk0 - dlnkinf) + kinf * Pr * Pr1 * dFdT;
            dkdM = k0 * dgdPr;
          }
          M = 1.0;
        }
      }
      sc[O_Q + r] = M * k * net;
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
    g.sync();
  }

  // wdot_k (k < K) by the padded ELL of species k (branch-free)
  __device__ static double wdot_k(const double* sc, int k) {
    double w0 = 0.0, w1 = 0.0;
#pragma unroll 4
    for (int m = 0; m + 1 < ELL; m += 2) {
      w0 = fma(T::ell_nu()[m * K + k], sc[O_Q + T::ell_r()[m * K + k]], w0);
      w1 = fma(T::ell_nu()[(m + 1) * K + k], sc[O_Q + T::ell_r()[(m + 1) * K + k]], w1);
    }
    if (ELL & 1) w0 = fma(T::ell_nu()[(ELL - 1) * K + k], sc[O_Q + T::ell_r()[(ELL - 1) * K + k]], w0);
    return w0 + w1;
  }

  // f = R(y) for the group's cell (this lane's components); rho: the cell's density; sc: SG doubles
  __device__ static int rhs(const Grp<G>& g, const double (&y)[R], double rho, double (&f)[R], double* sc) {
    double Tt, lnT, invT;
#pragma unroll
    for (int r = 0; r < R; ++r) f[r] = 0.0;
    if (species(g, y, rho, sc, Tt, lnT, invT)) return 1;
    reactions<false>(g, sc, nullptr, Tt, lnT, invT);
    double cvp = 0.0, up = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k = g.lane + G * r;
      if (k < K) {
        const double w = wdot_k(sc, k);
        f[r] = T::W()[k] * w / rho;
        cvp += sc[O_Y + k] * (sc[O_CP + k] - 1.0) * RU * T::invW()[k];
        up += (sc[O_H + k] - 1.0) * RU * Tt * w;
      }
    }
    const double cv = g.sum(cvp), su = g.sum(up);
    constexpr int rT = K / G;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r == rT && g.lane == K - G * rT) f[r] = -su / (rho * cv);
    g.sync();
    return 0;
  }

  // Analytic Jacobian of the group's cell: row i = lane + G r goes to J[i * ld + j * cs] (j = 0..N-1);
  // J is this group's (shared or global) matrix.  sc: SG scratch doubles, js: JG scratch doubles.
  __device__ static int jac(const Grp<G>& g, const double (&y)[R], double rho, double* J, long long ld, long long cs,
                            double* sc, double* js) {
    double Tt, lnT, invT;
    if (species(g, y, rho, sc, Tt, lnT, invT)) return 1;
    reactions<true>(g, sc, js, Tt, lnT, invT);
    const double* dr = js + J_DR;
    const double* dp = js + J_DP;
    double cvp = 0.0, up = 0.0, dcvp = 0.0, cvw = 0.0;
    double uoW[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k = g.lane + G * r;
      uoW[r] = 0.0;
      if (k >= N) continue;
      double* row = J + (long long)k * ld;
      for (int j = 0; j < N; ++j) row[j * cs] = 0.0;
      if (k >= K) continue;
      const double w = wdot_k(sc, k);
      const int len = T::ell_len()[k];
      double dT = 0.0;
      for (int m = 0; m < len; ++m) {
        const int rx = T::ell_r()[m * K + k];
        const double nu = T::ell_nu()[m * K + k];
        int s;
        s = T::reac0()[rx]; row[s * cs] = fma(nu, dr[rx], row[s * cs]);
        s = T::reac1()[rx]; if (s >= 0) row[s * cs] = fma(nu, dr[NR + rx], row[s * cs]);
        s = T::reac2()[rx]; if (s >= 0) row[s * cs] = fma(nu, dr[2 * NR + rx], row[s * cs]);
        s = T::prod0()[rx]; row[s * cs] = fma(nu, dp[rx], row[s * cs]);
        s = T::prod1()[rx]; if (s >= 0) row[s * cs] = fma(nu, dp[NR + rx], row[s * cs]);
        s = T::prod2()[rx]; if (s >= 0) row[s * cs] = fma(nu, dp[2 * NR + rx], row[s * cs]);
        dT = fma(nu, js[J_DT + rx], dT);
      }
      // third-body / falloff [M] dependence: dense in the collision partners
#pragma unroll 1
      for (int t = 0; t < NTB; ++t) {
        const double coef = T::nu_tb()[t * K + k] * js[J_DM + T::tb_rxn()[t]];
        if (coef != 0.0) {
          const double* e = T::eff() + t * K;
          for (int j = 0; j < K; ++j) row[j * cs] = fma(coef, e[j], row[j * cs]);
        }
      }
      const double Wk = T::W()[k];
      for (int j = 0; j < K; ++j) row[j * cs] = row[j * cs] * (Wk * T::invW()[j]);
      row[K * cs] = Wk * dT / rho;
      const double Y = sc[O_Y + k], iW = T::invW()[k];
      const double u = (sc[O_H + k] - 1.0) * RU * Tt;
      cvp += Y * (sc[O_CP + k] - 1.0) * RU * iW;
      up += u * w;
      const double* a = (Tt < T::Tmid()[k]) ? T::nasa_lo() : T::nasa_hi();
      const double dcp =
          fma(Tt, fma(Tt, fma(Tt, 4.0 * a[4 * K + k], 3.0 * a[3 * K + k]), 2.0 * a[2 * K + k]), a[K + k]);
      dcvp += Y * dcp * RU * iW;
      cvw += (sc[O_CP + k] - 1.0) * RU * w;
      uoW[r] = u * iW;
    }
    g.sync();
    // temperature row: f_T = -sum_k u_k wdot_k / (rho cv)
    const double cv = g.sum(cvp), su = g.sum(up), dcv = g.sum(dcvp), scw = g.sum(cvw);
    const double fT0 = -su / (rho * cv);
    const double icv = 1.0 / cv;
    constexpr int rT = K / G;
    const bool ownT = g.lane == K - G * rT;
    double* rowT = J + (long long)K * ld;
    for (int j = 0; j < N; ++j) {
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = g.lane + G * r;
        if (k < K) v += uoW[r] * J[(long long)k * ld + j * cs];
      }
      const double s = g.sum(v);
      if (ownT) {
        if (j < K) {
          const double cvj = (sc[O_CP + j] - 1.0) * RU * T::invW()[j];
          rowT[j * cs] = -s * icv - fT0 * cvj * icv;
        } else {
          rowT[j * cs] = -scw / (rho * cv) - s * icv - fT0 * dcv * icv;
        }
      }
    }
    g.sync();
    return 0;
  }
};

}  // namespace bdfb
