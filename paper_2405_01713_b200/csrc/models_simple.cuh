// models_simple.cuh -- device RHS/Jacobian for the small models, one cell per
// thread (G = 1).  Each model provides N, G, DIAG, BLOCK, SCRATCH, Params,
// rhs() and (dense models) jac() writing its rows with mat<N,G>().
//
// rhs() returns 0, or 1 for a recoverable failure (group-uniform); f must be
// 0 in register slots that hold no component.
#pragma once
#include "grp.cuh"
#include "lu.cuh"

namespace bdfb {

// y' = lambda y  (n = 1; the closed-form pin model)
struct ModelLinear {
  static constexpr int N = 1, G = 1, BLOCK = 128, SCRATCH = 0, MINB = 1;
  static constexpr bool DIAG = false;
  struct Params { double lambda; };
  __device__ static int rhs(const Grp<1>&, const Params& p, double, const double (&y)[1], double (&f)[1], double,
                            double*) {
    f[0] = p.lambda * y[0];
    return 0;
  }
  static constexpr int JSCRATCH = 0;
  __device__ static int jac(const Grp<1>& g, const Params& p, double, const double (&)[1], double, double* J,
                            double*, double*) {
    mat<1, 1>(J, g, 0, 0) = p.lambda;
    return 0;
  }
};

// Robertson stiff kinetics, k = (0.04, 3e7, 1e4)
struct ModelRobertson {
  static constexpr int N = 3, G = 1, BLOCK = 128, SCRATCH = 0, MINB = 1;
  static constexpr bool DIAG = false;
  struct Params { double k[3]; };
  __device__ static int rhs(const Grp<1>&, const Params& p, double, const double (&y)[3], double (&f)[3], double,
                            double*) {
    const double r1 = p.k[0] * y[0], r2 = p.k[1] * y[1] * y[1], r3 = p.k[2] * y[1] * y[2];
    f[0] = -r1 + r3;
    f[1] = r1 - r3 - r2;
    f[2] = r2;
    return 0;
  }
  static constexpr int JSCRATCH = 0;
  __device__ static int jac(const Grp<1>& g, const Params& p, double, const double (&y)[3], double, double* J,
                            double*, double*) {
    mat<3, 1>(J, g, 0, 0) = -p.k[0];
    mat<3, 1>(J, g, 0, 1) = p.k[2] * y[2];
    mat<3, 1>(J, g, 0, 2) = p.k[2] * y[1];
    mat<3, 1>(J, g, 1, 0) = p.k[0];
    mat<3, 1>(J, g, 1, 1) = -p.k[2] * y[2] - 2.0 * p.k[1] * y[1];
    mat<3, 1>(J, g, 1, 2) = -p.k[2] * y[1];
    mat<3, 1>(J, g, 2, 0) = 0.0;
    mat<3, 1>(J, g, 2, 1) = 2.0 * p.k[1] * y[1];
    mat<3, 1>(J, g, 2, 2) = 0.0;
    return 0;
  }
};

// Nyx-style optically thin H/He heating and cooling in ionisation equilibrium
// (the scalar ODE de/dt = R(e) + F of P:242; reading R21, the
// KWH96-form rate set restated in SURVEY.md Appendix B).  Linear solver:
// CVDiag.  n_e from the same regula-falsi rule as the reading:
// Illinois on [1e-12, 1 + 2 y_He], |dx| <= 1e-12 (1 + 2 y_He), <= 60 iters.
struct ModelNyxKwh {
  static constexpr int N = 1, G = 1, BLOCK = 128, SCRATCH = 0, MINB = 1;
  static constexpr bool DIAG = true;
  struct Params {
    double z, X, Y, gamma_ad;
    double gph[3], eph[3];
  };
  static constexpr double MP = 1.67262192369e-24, KB = 1.380649e-16;

  struct Pop { double T, nH0, nHp, nHe0, nHep, nHepp, ne, g; };

  __device__ static void eval(const Params& q, double e, double nH, double yHe, double xe, Pop& P) {
    const double mu = (1.0 + 4.0 * yHe) / (1.0 + yHe + xe);
    const double T = (q.gamma_ad - 1.0) * mu * MP * e / KB;
    const double sT = sqrt(T);
    const double T3 = T / 1e3, T5 = T / 1e5, T6 = T / 1e6;
    const double S5 = 1.0 / (1.0 + sqrt(T5));
    const double rfac = pow(T3, -0.2) / (1.0 + pow(T6, 0.7));
    const double aHp = 8.40e-11 / sT * rfac;
    const double aHep = 1.50e-10 * pow(T, -0.6353);
    const double ad = 1.9e-3 * pow(T, -1.5) * exp(-470000.0 / T) * (1.0 + 0.3 * exp(-94000.0 / T));
    const double aHepp = 3.36e-10 / sT * rfac;
    const double GeH0 = 5.85e-11 * sT * exp(-157809.1 / T) * S5;
    const double GeHe0 = 2.38e-11 * sT * exp(-285335.4 / T) * S5;
    const double GeHep = 5.68e-12 * sT * exp(-631515.0 / T) * S5;
    const double ne = xe * nH;
    const double nH0 = nH * aHp / (aHp + GeH0 + q.gph[0] / ne);
    const double nHp = nH - nH0;
    const double ion0 = GeHe0 + q.gph[1] / ne;
    const double ion1 = GeHep + q.gph[2] / ne;
    const double nHep = yHe * nH / (1.0 + (aHep + ad) / ion0 + ion1 / aHepp);
    const double nHe0 = nHep * (aHep + ad) / ion0;
    const double nHepp = nHep * ion1 / aHepp;
    P.T = T; P.nH0 = nH0; P.nHp = nHp; P.nHe0 = nHe0; P.nHep = nHep; P.nHepp = nHepp; P.ne = ne;
    P.g = xe - (nHp + nHep + 2.0 * nHepp) / nH;
  }

  __device__ static int rhs(const Grp<1>&, const Params& q, double, const double (&y)[1], double (&f)[1],
                            double rho, double*) {
    const double e = y[0];
    f[0] = 0.0;
    const double nH = q.X * rho / MP;
    const double yHe = q.Y / (4.0 * q.X);
    const double xmax = 1.0 + 2.0 * yHe;
    if (!(e > 0.0) || !isfinite(e)) return 1;
    const double Tmax = (q.gamma_ad - 1.0) * ((1.0 + 4.0 * yHe) / (1.0 + yHe + 1e-12)) * MP * e / KB;
    const double Tmin = (q.gamma_ad - 1.0) * ((1.0 + 4.0 * yHe) / (1.0 + yHe + xmax)) * MP * e / KB;
    if (Tmin < 1.0 || Tmax > 1e9) return 1;
    Pop A, B, Cc;
    double a = 1e-12, b = xmax;
    eval(q, e, nH, yHe, a, A);
    eval(q, e, nH, yHe, b, B);
    double fa = A.g, fb = B.g;
    if (fb == 0.0) {
      Cc = B;
    } else if (fa >= 0.0) {
      Cc = A;
    } else {
      const double tol = 1e-12 * xmax;
      double cprev = 0.0;
      int side = 0;
      for (int it = 0; it < 60; ++it) {
        const double c = (a * fb - b * fa) / (fb - fa);
        eval(q, e, nH, yHe, c, Cc);
        const double fc = Cc.g;
        if (it > 0 && fabs(c - cprev) <= tol) break;
        cprev = c;
        if (fc == 0.0) break;
        if ((fc > 0.0) == (fb > 0.0)) {
          b = c; fb = fc;
          if (side == -1) fa *= 0.5;
          side = -1;
        } else {
          a = c; fa = fc;
          if (side == +1) fb *= 0.5;
          side = +1;
        }
      }
    }
    const double T = Cc.T, sT = sqrt(T);
    const double T3 = T / 1e3, T5 = T / 1e5, T6 = T / 1e6;
    const double S5 = 1.0 / (1.0 + sqrt(T5));
    const double ne = Cc.ne;
    const double rec = pow(T3, -0.2) / (1.0 + pow(T6, 0.7));
    double L = 0.0;
    L += 7.50e-19 * exp(-118348.0 / T) * S5 * ne * Cc.nH0;
    L += 5.54e-17 * pow(T, -0.397) * exp(-473638.0 / T) * S5 * ne * Cc.nHep;
    L += 1.27e-21 * sT * exp(-157809.1 / T) * S5 * ne * Cc.nH0;
    L += 9.38e-22 * sT * exp(-285335.4 / T) * S5 * ne * Cc.nHe0;
    L += 4.95e-22 * sT * exp(-631515.0 / T) * S5 * ne * Cc.nHep;
    L += 8.70e-27 * sT * rec * ne * Cc.nHp;
    L += 1.55e-26 * pow(T, 0.3647) * ne * Cc.nHep;
    L += 3.48e-26 * sT * rec * ne * Cc.nHepp;
    L += 1.24e-13 * pow(T, -1.5) * exp(-470000.0 / T) * (1.0 + 0.3 * exp(-94000.0 / T)) * ne * Cc.nHep;
    const double lt = 5.5 - log10(T);
    const double gff = 1.1 + 0.34 * exp(-lt * lt / 3.0);
    L += 1.42e-27 * gff * sT * (Cc.nHp + Cc.nHep + 4.0 * Cc.nHepp) * ne;
    const double zp1 = 1.0 + q.z;
    L += 5.41e-36 * ne * T * (zp1 * zp1 * zp1 * zp1);
    const double H = Cc.nH0 * q.eph[0] + Cc.nHe0 * q.eph[1] + Cc.nHep * q.eph[2];
    f[0] = (H - L) / rho;
    return 0;
  }
  static constexpr int JSCRATCH = 0;
  __device__ static int jac(const Grp<1>&, const Params&, double, const double (&)[1], double, double*, double*,
                            double*) {
    return -1;  // CVDiag model: no analytic Jacobian
  }
};

}  // namespace bdfb
