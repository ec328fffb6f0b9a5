// problem.cuh -- problem data evaluated on the device: exact / initial / Dirichlet values and the
// forcing of the manufactured solutions, derived from the strong form by forward-mode jets.
//
//  * 2D: paper Example 1 exact solution; "initial conditions, boundary conditions and
//    forcing terms can be derived from the analytical solutions".
//  * 3D: paper Example 2 exact solution, reflected into the BASELINE geometry
//    (porous [0,1]^3 below the conduit [0,1]^2 x [1,2], Gamma z = 1): z_paper = 1 - z,
//    u_z -> -u_z, pressures unchanged (C17).
//  * Injection (cfg2/cfg4): zero forcing and initial state, parabolic inflow of peak 1 on the top
//    conduit face, no-slip sides, p_i = 0 on dOmega_p \ Gamma (C16).
//  * Constant: p_i = c, u = 0, p = c / rho (an exact discrete steady state; invariant test).
//
// Forcing (strong form):
//   q_F = phi_F C_F dp_F/dt - (k_F/mu) lap p_F + sigma* k_f/mu (p_F - p_f)                 (1)
//   q_f = phi_f C_f dp_f/dt - (k_f/mu) lap p_f + sigma* k_f/mu (p_f - p_F) + sigma k_m/mu (p_f - p_m)  (2)
//   q_m = phi_m C_m dp_m/dt - (k_m/mu) lap p_m + sigma k_m/mu (p_m - p_f)                   (3)
//   f_a = du_a/dt - nu (lap u_a + d_a div u) + d_a p + (u . grad) u_a                       (4)
// (div T = nu (lap u + grad div u) - grad p for T = 2 nu D(u) - p I.)
#pragma once
#include "common.cuh"

namespace lp {

enum { PROB_MMS = 0, PROB_INJECTION = 1, PROB_CONSTANT = 2, PROB_MMS_STEADY = 3 };

struct Coef {
  double phiC[3];  // phi_i C_i, index 0 m, 1 f, 2 F
  double k[3];     // permeabilities
  double sigma, sigma_star, mu, nu, rho, alpha, eta;
};

struct ProbData {
  int kind;
  double peak;   // injection inflow peak
  double cval;   // constant problem value
};

// Exact fields as jets: P[0] = p_m, P[1] = p_f, P[2] = p_F, U[0..D-1], Pc = conduit pressure.
template <int D>
HD void mms_jets(const double* x, double t, Jet P[3], Jet U[3], Jet& Pc) {
  const double pi = 3.14159265358979323846;
  if (D == 2) {
    Jet X = jvar(x[0], 0), Y = jvar(x[1], 1), T = jvar(t, 3);
    Jet ct = jcos(T);
    Jet a = 2.0 - pi * jsin(pi * X);
    Jet Y2 = Y * Y;
    P[0] = a * jsin(0.5 * pi * (3.0 * Y2 * Y - 2.0 * Y2)) * ct;
    P[1] = a * jcos(pi * (1.0 - Y)) * ct;
    P[2] = a * (1.0 - Y - jcos(pi * Y)) * ct;
    Jet ym = Y - 1.0;
    U[0] = (X * X * ym * ym + Y) * ct;
    U[1] = ((-2.0 / 3.0) * X * ym * ym * ym + a) * ct;
    U[2] = jconst(0.0);
    Pc = a * jsin(0.5 * pi * Y) * ct;
  } else {
    Jet X = jvar(x[0], 0), Y = jvar(x[1], 1), Z = jvar(x[2], 2), T = jvar(t, 3);
    Jet zp = 1.0 - Z;  // z of the paper
    Jet e = jexp(-T);
    Jet XY = X * Y;
    Jet sxy = jsin(XY), cxy = jcos(XY);
    Jet r2 = X * X + Y * Y;
    Jet cz = jcos(zp);
    P[0] = -zp + jexp(zp) - e * sxy * cz;
    P[1] = P[0];
    P[2] = -zp + (8.0 - r2) * e * sxy * cz;
    U[0] = (2.0 * X * sxy + Y * (r2 - 8.0) * cxy) * e;
    U[1] = (2.0 * Y * sxy + X * (r2 - 8.0) * cxy) * e;
    Jet uzp = 1.0 + (r2 * (r2 - 8.0) * sxy - 4.0 * sxy - 8.0 * XY * cxy) * zp * e;
    U[2] = -uzp;
    Jet s2 = r2 + zp * zp;
    Pc = (-16.0 * XY * cxy + (s2 - 8.0) * (2.0 * s2 - 1.0) * sxy - 8.0 * sxy) * e;
  }
}

template <int D>
HD double jlap(const Jet& J) {
  double s = 0.0;
  for (int a = 0; a < D; ++a) s += J.H[a][a];
  return s;
}

// Porous values (m, f, F) at x, time t.
template <int D>
HD void porous_values(const ProbData& pd, const double* x, double t, double out[3]) {
  if (pd.kind == PROB_MMS || pd.kind == PROB_MMS_STEADY) {
    Jet P[3], U[3], Pc;
    mms_jets<D>(x, pd.kind == PROB_MMS_STEADY ? 0.0 : t, P, U, Pc);
    for (int i = 0; i < 3; ++i) out[i] = P[i].v;
  } else if (pd.kind == PROB_CONSTANT) {
    for (int i = 0; i < 3; ++i) out[i] = pd.cval;
  } else {
    for (int i = 0; i < 3; ++i) out[i] = 0.0;
  }
}

// Porous forcing (m, f, F) at x, time t (eqs. (1)-(3)).
template <int D>
HD void porous_forcing(const ProbData& pd, const Coef& co, const double* x, double t, double q[3]) {
  if (pd.kind == PROB_MMS || pd.kind == PROB_MMS_STEADY) {
    Jet P[3], U[3], Pc;
    const bool steady = pd.kind == PROB_MMS_STEADY;
    mms_jets<D>(x, steady ? 0.0 : t, P, U, Pc);
    const double sFf = co.sigma_star * co.k[1] / co.mu, sfm = co.sigma * co.k[0] / co.mu;
    double dt[3];
    for (int i = 0; i < 3; ++i) dt[i] = steady ? 0.0 : P[i].g[3];
    q[2] = co.phiC[2] * dt[2] - co.k[2] / co.mu * jlap<D>(P[2]) + sFf * (P[2].v - P[1].v);
    q[1] = co.phiC[1] * dt[1] - co.k[1] / co.mu * jlap<D>(P[1]) + sFf * (P[1].v - P[2].v) +
           sfm * (P[1].v - P[0].v);
    q[0] = co.phiC[0] * dt[0] - co.k[0] / co.mu * jlap<D>(P[0]) + sfm * (P[0].v - P[1].v);
  } else {
    q[0] = q[1] = q[2] = 0.0;
  }
}

// Conduit velocity (Dirichlet / initial / exact) at x; on_top = node on the inflow face (injection).
template <int D>
HD void velocity_values(const ProbData& pd, const double* x, double t, bool on_top, double u[3]) {
  u[0] = u[1] = u[2] = 0.0;
  if (pd.kind == PROB_MMS || pd.kind == PROB_MMS_STEADY) {
    Jet P[3], U[3], Pc;
    mms_jets<D>(x, pd.kind == PROB_MMS_STEADY ? 0.0 : t, P, U, Pc);
    for (int a = 0; a < D; ++a) u[a] = U[a].v;
  } else if (pd.kind == PROB_INJECTION && on_top) {
    double prof = 1.0;
    for (int a = 0; a < D - 1; ++a) prof *= 4.0 * x[a] * (1.0 - x[a]);
    u[D - 1] = -pd.peak * prof;
  }
}

template <int D>
HD double pressure_value(const ProbData& pd, const Coef& co, const double* x, double t) {
  if (pd.kind == PROB_MMS || pd.kind == PROB_MMS_STEADY) {
    Jet P[3], U[3], Pc;
    mms_jets<D>(x, pd.kind == PROB_MMS_STEADY ? 0.0 : t, P, U, Pc);
    return Pc.v;
  }
  if (pd.kind == PROB_CONSTANT) return pd.cval / co.rho;
  return 0.0;
}

// Momentum forcing f (eq. (4)).
template <int D>
HD void velocity_forcing(const ProbData& pd, const Coef& co, const double* x, double t, double f[3]) {
  f[0] = f[1] = f[2] = 0.0;
  if (pd.kind != PROB_MMS && pd.kind != PROB_MMS_STEADY) return;
  Jet P[3], U[3], Pc;
  const bool steady = pd.kind == PROB_MMS_STEADY;
  mms_jets<D>(x, steady ? 0.0 : t, P, U, Pc);
  for (int a = 0; a < D; ++a) {
    double lap = jlap<D>(U[a]);
    double graddiv = 0.0;
    for (int b = 0; b < D; ++b) graddiv += U[b].H[a][b];
    double conv = 0.0;
    for (int b = 0; b < D; ++b) conv += U[b].v * U[a].g[b];
    f[a] = (steady ? 0.0 : U[a].g[3]) - co.nu * (lap + graddiv) + Pc.g[a] + conv;
  }
}

}  // namespace lp
