// tables.h -- host construction of the Kuhn simplex tables and the P2/P1 barycentric reference
// tensors (setup work of lpfem_create, stage a0).
//
// The reference tensors integrate products of P2 Lagrange basis functions in barycentric form,
//   vertex i: lam_i (2 lam_i - 1),  edge (a,b): 4 lam_a lam_b,
// and their lam-derivatives (treating lam_0..lam_D as independent; the chain rule with
// grad lam_k is then exact because sum_k grad lam_k = 0).  Integration uses the Duffy map of the
// unit cube onto the simplex with a 4-point Gauss-Legendre rule per axis: exact for polynomials of
// degree <= 7 in each collapsed variable, i.e. for every integrand of the weak form (degree <= 5,
// P:168-213), so the discrete operators are independent of any quadrature choice (C13).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace lp {

inline void build_kuhn(int D, KuhnTables& T) {
  std::memset(&T, 0, sizeof(T));
  std::memset(T.lookup, -1, sizeof(T.lookup));
  int perm[3] = {0, 1, 2};
  int t = 0;
  do {  // permutations in lexicographic order
    for (int a = 0; a < D; ++a) {
      T.perm[t][a] = perm[a];
      T.pos[t][perm[a]] = a;
    }
    int V[4][3] = {};
    for (int k = 1; k <= D; ++k) {
      for (int a = 0; a < D; ++a) V[k][a] = V[k - 1][a];
      V[k][perm[k - 1]] += 2;
    }
    int i = 0;
    for (int k = 0; k <= D; ++k, ++i)
      for (int a = 0; a < D; ++a) T.off[t][i][a] = (signed char)V[k][a];
    int e = 0;
    for (int a = 0; a <= D; ++a)
      for (int b = a + 1; b <= D; ++b, ++i, ++e) {
        for (int c = 0; c < D; ++c) T.off[t][i][c] = (signed char)((V[a][c] + V[b][c]) / 2);
        T.edge[e][0] = a;
        T.edge[e][1] = b;
      }
    for (int j = 0; j < i; ++j) {
      int code = 0, s = 1;
      for (int a = 0; a < D; ++a, s *= 3) code += T.off[t][j][a] * s;
      T.lookup[t][code] = (signed char)j;
    }
    ++t;
  } while (std::next_permutation(perm, perm + D));
}

// Duffy-mapped Gauss-Legendre points on the D-simplex: barycentrics and weights normalised so that
// sum w = 1 (i.e. the rule computes (1/|K|) int_K).
inline void simplex_rule(int D, std::vector<std::vector<double>>& lam, std::vector<double>& w) {
  const double s1 = std::sqrt(3.0 / 7.0 - 2.0 / 7.0 * std::sqrt(6.0 / 5.0));
  const double s2 = std::sqrt(3.0 / 7.0 + 2.0 / 7.0 * std::sqrt(6.0 / 5.0));
  const double w1 = (18.0 + std::sqrt(30.0)) / 36.0, w2 = (18.0 - std::sqrt(30.0)) / 36.0;
  const double gx[4] = {0.5 * (1 - s2), 0.5 * (1 - s1), 0.5 * (1 + s1), 0.5 * (1 + s2)};
  const double gw[4] = {0.5 * w2, 0.5 * w1, 0.5 * w1, 0.5 * w2};
  lam.clear();
  w.clear();
  if (D == 0) {
    lam.push_back({1.0});
    w.push_back(1.0);
    return;
  }
  int n = 1;
  for (int a = 0; a < D; ++a) n *= 4;
  for (int q = 0; q < n; ++q) {
    int id[3] = {q % 4, (q / 4) % 4, (q / 16) % 4};
    double u = gx[id[0]], v = D > 1 ? gx[id[1]] : 0.0, z = D > 2 ? gx[id[2]] : 0.0;
    double xi[3] = {0, 0, 0}, jac = 1.0, wt = gw[id[0]];
    if (D == 1) {
      xi[0] = u;
    } else if (D == 2) {
      xi[0] = u;
      xi[1] = (1 - u) * v;
      jac = 2.0 * (1 - u);
      wt *= gw[id[1]];
    } else {
      xi[0] = u;
      xi[1] = (1 - u) * v;
      xi[2] = (1 - u) * (1 - v) * z;
      jac = 6.0 * (1 - u) * (1 - u) * (1 - v);
      wt *= gw[id[1]] * gw[id[2]];
    }
    std::vector<double> l(D + 1);
    double s = 0.0;
    for (int a = 0; a < D; ++a) {
      l[a + 1] = xi[a];
      s += xi[a];
    }
    l[0] = 1.0 - s;
    lam.push_back(l);
    w.push_back(wt * jac);
  }
}

// P2 basis values and lam-derivatives at barycentric point l (D+1 entries).
inline void p2_eval(int D, const std::vector<double>& l, double* phi, double dphi[][4]) {
  int n = 0;
  for (int i = 0; i <= D; ++i, ++n) {
    phi[n] = l[i] * (2.0 * l[i] - 1.0);
    for (int k = 0; k <= D; ++k) dphi[n][k] = (k == i) ? 4.0 * l[i] - 1.0 : 0.0;
  }
  for (int a = 0; a <= D; ++a)
    for (int b = a + 1; b <= D; ++b, ++n) {
      phi[n] = 4.0 * l[a] * l[b];
      for (int k = 0; k <= D; ++k) dphi[n][k] = (k == a ? 4.0 * l[b] : 0.0) + (k == b ? 4.0 * l[a] : 0.0);
    }
}

template <int D>
void build_ref(RefT<D>& R) {
  std::memset(&R, 0, sizeof(R));
  constexpr int N = n2_of(D), L = D + 1;
  std::vector<std::vector<double>> lam;
  std::vector<double> w;
  simplex_rule(D, lam, w);
  for (size_t q = 0; q < w.size(); ++q) {
    double phi[10], dphi[10][4];
    p2_eval(D, lam[q], phi, dphi);
    const double wq = w[q];
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        R.M22[i][j] += wq * phi[i] * phi[j];
        for (int k = 0; k < L; ++k)
          for (int l = 0; l < L; ++l) R.G22[i][k][j][l] += wq * dphi[i][k] * dphi[j][l];
        for (int m = 0; m < N; ++m)
          for (int l = 0; l < L; ++l) R.C3[i][m][j][l] += wq * phi[i] * phi[m] * dphi[j][l];
      }
    for (int m = 0; m < L; ++m)
      for (int j = 0; j < N; ++j)
        for (int l = 0; l < L; ++l) R.D12[m][j][l] += wq * lam[q][m] * dphi[j][l];
  }
  // facet tensors on the (D-1)-simplex
  constexpr int NF = n2_of(D - 1), LF = D;
  simplex_rule(D - 1, lam, w);
  for (size_t q = 0; q < w.size(); ++q) {
    double phi[10], dphi[10][4];
    p2_eval(D - 1, lam[q], phi, dphi);
    for (int i = 0; i < NF; ++i)
      for (int j = 0; j < NF; ++j) {
        R.MF[i][j] += w[q] * phi[i] * phi[j];
        for (int l = 0; l < LF; ++l) R.TF[i][j][l] += w[q] * phi[i] * dphi[j][l];
      }
  }
}

}  // namespace lp
