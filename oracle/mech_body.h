/*
 * mech_body.h -- constant-volume, constant-internal-energy reactor RHS, the
 * oracle's plain transcription of SURVEY.md §8(c).6 (C3-C5; the paper's 0-D
 * reactor "assumed constant internal energy"; split form chemODE
 * dU/dt = F + R with F frozen over dt_CFD).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Included twice by models.c: once
 * with RT = double (the RHS itself) and once with RT = double complex (the
 * complex-step Jacobian, J[:,j] = Im f(y + i*eps*e_j)/eps, §8c.4).
 *
 * Required macros: RT, FN(name), EXPF, LOGF, REALPART.
 */

static int FN(mech_rhs)(const orc_problem *p, const RT *y, RT *f, double *scale)
{
  const orc_mech *m = p->mech;
  const int K = m->K;
  const double Rc = 1.98720425864083;      /* cal/(mol K), for Ea        */
  const double Ru = 8.31446261815324e7;    /* erg/(mol K), for Kc, u, cv */
  const double patm = 1013250.0;           /* dyn/cm^2                   */
  const double rho = p->rho;

  RT C[ORC_NMAX], cpR[ORC_NMAX], hRT[ORC_NMAX], gRT[ORC_NMAX], wdot[ORC_NMAX];
  double wabs[ORC_NMAX];          /* sum_r |nu_rk| (|fwd_r| + |rvs_r|): reading R19 scale */
  RT T = y[K];
  if (!(REALPART(T) > 0.0)) return 1;
  RT lnT = LOGF(T);
  RT invT = 1.0 / T;

  for (int k = 0; k < K; ++k) C[k] = rho * y[k] / m->W[k];

  /* NASA-7 polynomials: cp/R, h/RT, s/R; g/RT = h/RT - s/R */
  for (int k = 0; k < K; ++k) {
    const double *c = m->nasa + 15 * k;
    const double *a = (REALPART(T) < c[0]) ? c + 1 : c + 8;
    RT T2 = T * T, T3 = T2 * T, T4 = T3 * T;
    cpR[k] = a[0] + a[1] * T + a[2] * T2 + a[3] * T3 + a[4] * T4;
    hRT[k] = a[0] + a[1] * T / 2.0 + a[2] * T2 / 3.0 + a[3] * T3 / 4.0
           + a[4] * T4 / 5.0 + a[5] * invT;
    RT sR = a[0] * lnT + a[1] * T + a[2] * T2 / 2.0 + a[3] * T3 / 3.0
          + a[4] * T4 / 4.0 + a[6];
    gRT[k] = hRT[k] - sR;
    wdot[k] = 0.0;
    wabs[k] = 0.0;
  }

  for (int r = 0; r < m->nr; ++r) {
    const double *ar = m->arr + 3 * r;
    /* k_f = A T^beta exp(-Ea/(Rc T)) */
    RT kf = EXPF(log(ar[0]) + ar[1] * lnT - (ar[2] / Rc) * invT);
    int ty = m->type[r];
    if (ty >= 1) {
      RT M = 0.0;
      for (int k = 0; k < K; ++k) M = M + m->eff[r * K + k] * C[k];
      if (ty == 1) {
        kf = kf * M;                       /* plain third body          */
      } else {
        const double *a0 = m->arr0 + 3 * r;
        RT k0 = EXPF(log(a0[0]) + a0[1] * lnT - (a0[2] / Rc) * invT);
        RT Pr = k0 * M / kf;
        RT F = 1.0;                        /* Lindemann                 */
        if (ty == 3) {                     /* Troe                      */
          const double *tr = m->troe + 4 * r;
          RT Fc = (1.0 - tr[0]) * EXPF(-T / tr[1]) + tr[0] * EXPF(-T / tr[2]);
          if (m->has_t2[r]) Fc = Fc + EXPF(-tr[3] * invT);
          RT lFc = LOGF(Fc) / log(10.0);
          RT cc = -0.4 - 0.67 * lFc;
          RT nn = 0.75 - 1.27 * lFc;
          RT lPr = LOGF(Pr) / log(10.0);
          RT f1 = (lPr + cc) / (nn - 0.14 * (lPr + cc));
          RT lF = lFc / (1.0 + f1 * f1);
          F = EXPF(lF * log(10.0));
        }
        kf = kf * (Pr / (1.0 + Pr)) * F;
      }
    }
    RT fwd = kf;
    for (int s = 0; s < 3; ++s) {
      int k = m->reac[3 * r + s];
      if (k >= 0) fwd = fwd * C[k];
    }
    RT q = fwd;
    double qabs = REALPART(fwd) < 0 ? -REALPART(fwd) : REALPART(fwd);
    if (m->rev[r]) {
      RT sg = 0.0;
      int dnu = 0;
      for (int s = 0; s < 3; ++s) {
        int k = m->prod[3 * r + s];
        if (k >= 0) { sg = sg + gRT[k]; dnu += 1; }
      }
      for (int s = 0; s < 3; ++s) {
        int k = m->reac[3 * r + s];
        if (k >= 0) { sg = sg - gRT[k]; dnu -= 1; }
      }
      /* Kc = Kp (patm/(R T))^dnu,  Kp = exp(-sum nu g/RT) */
      RT Kc = EXPF(-sg);
      RT cfac = patm / (Ru * T);
      for (int d = 0; d < dnu; ++d) Kc = Kc * cfac;
      for (int d = 0; d < -dnu; ++d) Kc = Kc / cfac;
      RT rvs = kf / Kc;
      for (int s = 0; s < 3; ++s) {
        int k = m->prod[3 * r + s];
        if (k >= 0) rvs = rvs * C[k];
      }
      q = fwd - rvs;
      qabs += REALPART(rvs) < 0 ? -REALPART(rvs) : REALPART(rvs);
    }
    for (int s = 0; s < 3; ++s) {
      int k = m->reac[3 * r + s];
      if (k >= 0) { wdot[k] = wdot[k] - q; wabs[k] += qabs; }
    }
    for (int s = 0; s < 3; ++s) {
      int k = m->prod[3 * r + s];
      if (k >= 0) { wdot[k] = wdot[k] + q; wabs[k] += qabs; }
    }
  }

  /* dY_k/dt = W_k wdot_k / rho + F_Yk */
  RT cv = 0.0, su = 0.0;
  for (int k = 0; k < K; ++k) {
    f[k] = m->W[k] * wdot[k] / rho;
    cv = cv + y[k] * (cpR[k] - 1.0) * Ru / m->W[k];
    su = su + (hRT[k] - 1.0) * Ru * T * wdot[k];
  }
  /* dT/dt = -sum_k u_k wdot_k / (rho cv) + F_T */
  f[K] = -su / (rho * cv);
  if (scale) {
    double st = 0.0, cvr = REALPART(cv);
    for (int k = 0; k < K; ++k) {
      scale[k] = m->W[k] * wabs[k] / rho;
      double u = (REALPART(hRT[k]) - 1.0) * Ru * REALPART(T);
      st += (u < 0 ? -u : u) * wabs[k];
    }
    scale[K] = st / (rho * (cvr < 0 ? -cvr : cvr));
    if (p->fext)
      for (int k = 0; k <= K; ++k) scale[k] += p->fext[k] < 0 ? -p->fext[k] : p->fext[k];
  }
  if (p->fext) for (int k = 0; k <= K; ++k) f[k] = f[k] + p->fext[k];
  return 0;
}
