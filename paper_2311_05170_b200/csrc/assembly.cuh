// assembly.cuh -- sparsity patterns, operator assembly, prolongation, right-hand sides and
// write-back on structured Kuhn boxes.  All kernels are row-gather: one thread owns one matrix
// row (or one node), walks the simplices around its node and accumulates into its own row, so
// assembly is atomic-free and deterministic without colouring.
//
// Operators (weak form P:168-213, eq. CoupledFormu; Algorithm 3):
//   porous  A_F = c_F M + K[k_F/mu] + M[sigma* k_f/mu]
//           A_f = c_f M + K[k_f/mu] + M[(sigma k_m + sigma* k_f)/mu]
//           A_m = c_m M + K[k_m/mu] + M[sigma k_m/mu]             c_i = phi_i C_i / dt
//   conduit (eta/dt) M_u + 2 nu eta (D u, D v) + (eta nu alpha/sqrt(k_F)) <P_tau u, P_tau v>_Gamma
//           + eta ((W.grad) u, v) [+ eta ((u.grad) U, v) for the Newton-linearised fine correction]
//           - eta (p, div v);   continuity  eta (q, div u)
// The permeabilities carry the per-coarse-cell multiplier (C15).
#pragma once
#include "common.cuh"
#include "problem.cuh"

namespace lp {

__constant__ KuhnTables c_kt[4];        // index = dimension (1..3)
__constant__ signed char c_nb[4][8][72][3];  // P2 neighbour offsets per parity class (sorted, lex)
__constant__ int c_nbn[4][8];
__constant__ signed char c_nb1[4][8][32][3]; // P1 neighbour vertices (half-grid offsets), sorted
__constant__ int c_nb1n[4][8];

struct Level {  // device view of one level of one region
  LevelGeom G;
  int m[3], core[3];  // subdomain grid and core cells per axis (fine level)
};

// ---------------------------------------------------------------------------------------------
// simplices around a node
template <int D, class F>
__device__ __forceinline__ void for_simplices_at(const int l[3], const int nc[3], F&& f) {
  int cand[3][2], ncand[3] = {1, 1, 1};
  for (int a = 0; a < D; ++a) {
    if (l[a] & 1) {
      cand[a][0] = (l[a] - 1) >> 1;
      ncand[a] = 1;
    } else {
      int k = 0;
      if ((l[a] >> 1) - 1 >= 0) cand[a][k++] = (l[a] >> 1) - 1;
      if ((l[a] >> 1) < nc[a]) cand[a][k++] = l[a] >> 1;
      ncand[a] = k;
    }
  }
  const int i2max = D > 2 ? ncand[2] : 1;
  const int i1max = D > 1 ? ncand[1] : 1;
  for (int i2 = 0; i2 < i2max; ++i2)
    for (int i1 = 0; i1 < i1max; ++i1)
      for (int i0 = 0; i0 < ncand[0]; ++i0) {
        int c[3] = {cand[0][i0], D > 1 ? cand[1][i1] : 0, D > 2 ? cand[2][i2] : 0};
        int code = 0, s = 1;
        for (int a = 0; a < D; ++a, s *= 3) code += (l[a] - 2 * c[a]) * s;
        for (int t = 0; t < nt_of(D); ++t) {
          int i = c_kt[D].lookup[t][code];
          if (i >= 0) f(c, t, i);
        }
      }
}

template <int D>
__device__ __forceinline__ int parity_class(const int l[3]) {
  int k = 0;
  for (int a = 0; a < D; ++a) k |= (l[a] & 1) << a;
  return k;
}

__device__ __forceinline__ long long find_slot(const int* __restrict__ col, long long lo, long long hi, int key) {
  // first position in [lo, hi) with col == key (binary search; rows sorted)
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (col[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------------------------
// patterns
template <int D>
__device__ __forceinline__ int count_nb(const int l[3], const int np[3]) {
  int k = parity_class<D>(l), n = 0;
  for (int q = 0; q < c_nbn[D][k]; ++q) {
    bool ok = true;
    for (int a = 0; a < D; ++a) {
      int v = l[a] + c_nb[D][k][q][a];
      ok = ok && v >= 0 && v < np[a];
    }
    n += ok;
  }
  return n;
}
template <int D>
__device__ __forceinline__ int count_nb1(const int l[3], const int np[3]) {
  int k = parity_class<D>(l), n = 0;
  for (int q = 0; q < c_nb1n[D][k]; ++q) {
    bool ok = true;
    for (int a = 0; a < D; ++a) {
      int v = l[a] + c_nb1[D][k][q][a];
      ok = ok && v >= 0 && v < np[a];
    }
    n += ok;
  }
  return n;
}

// row lengths.  family 0: scalar P2; family 1: Taylor-Hood saddle (velocity comps, then P1).
template <int D>
__global__ void k_pattern_count(const SysDesc* __restrict__ sys, int family, long long* __restrict__ cnt) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  int l[3] = {0, 0, 0};
  long long n;
  if (family == 0) {
    unlex<D>(r, S.np, l);
    n = count_nb<D>(l, S.np);
  } else if (r < D * S.n2) {
    unlex<D>(r % S.n2, S.np, l);
    n = (long long)D * count_nb<D>(l, S.np) + count_nb1<D>(l, S.np);
  } else {
    int shp1[3] = {S.nc[0] + 1, S.nc[1] + 1, S.nc[2] + 1};
    unlex<D>(r - D * S.n2, shp1, l);
    for (int a = 0; a < D; ++a) l[a] *= 2;
    n = (long long)D * count_nb<D>(l, S.np);
  }
  cnt[S.row_off + r] = n;
}

template <int D>
__global__ void k_pattern_fill(const SysDesc* __restrict__ sys, int family, const long long* __restrict__ rowptr,
                               int* __restrict__ col) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  long long p = rowptr[S.row_off + r];
  int l[3] = {0, 0, 0};
  int nblocks = 1;
  bool p1cols = false;
  if (family == 0) {
    unlex<D>(r, S.np, l);
  } else if (r < D * S.n2) {
    unlex<D>(r % S.n2, S.np, l);
    nblocks = D;
    p1cols = true;
  } else {
    int shp1[3] = {S.nc[0] + 1, S.nc[1] + 1, S.nc[2] + 1};
    unlex<D>(r - D * S.n2, shp1, l);
    for (int a = 0; a < D; ++a) l[a] *= 2;
    nblocks = D;
  }
  const int k = parity_class<D>(l);
  for (int b = 0; b < nblocks; ++b)
    for (int q = 0; q < c_nbn[D][k]; ++q) {
      int v[3];
      bool ok = true;
      for (int a = 0; a < D; ++a) {
        v[a] = l[a] + c_nb[D][k][q][a];
        ok = ok && v[a] >= 0 && v[a] < S.np[a];
      }
      if (ok) col[p++] = b * S.n2 + (int)lex<D>(v, S.np);
    }
  if (p1cols) {
    int shp1[3] = {S.nc[0] + 1, S.nc[1] + 1, S.nc[2] + 1};
    for (int q = 0; q < c_nb1n[D][k]; ++q) {
      int v[3];
      bool ok = true;
      for (int a = 0; a < D; ++a) {
        v[a] = l[a] + c_nb1[D][k][q][a];
        ok = ok && v[a] >= 0 && v[a] < S.np[a];
        v[a] >>= 1;
      }
      if (ok) col[p++] = D * S.n2 + (int)lex<D>(v, shp1);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// coefficient multiplier of the porous coarse cell containing box cell c (C15)
template <int D>
__device__ __forceinline__ double cell_mult(const double* __restrict__ kmult, const Level& L, const SysDesc& S,
                                            const int c[3], const int nH[3]) {
  if (!kmult) return 1.0;
  int cc[3];
  for (int a = 0; a < D; ++a) cc[a] = (S.c0[a] + c[a]) / L.G.R;
  return kmult[lex<D>(cc, nH)];
}

struct PorousCoefs {  // per field f (0 m, 1 f, 2 F): A_f = c M + s_e (kappa K + gamma M)
  double c[3], kappa[3], gamma[3];
  double gFf, gfm;      // exchange weights sigma* k_f/mu, sigma k_m/mu (times s_e)
};

// porous operators, unscaled values; also the diagonal.
template <int D>
__global__ void k_porous_assemble(const SysDesc* __restrict__ sys, Level L, PorousCoefs pc,
                                  const double* __restrict__ kmult, int nH0, int nH1, int nH2,
                                  const RefT<D>* __restrict__ ref, const long long* __restrict__ rowptr,
                                  const int* __restrict__ col, double* __restrict__ val, long long nnz_total,
                                  double* __restrict__ diag, long long rows_total) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  constexpr int N = n2_of(D);
  const int nH[3] = {nH0, nH1, nH2};
  int l[3] = {0, 0, 0};
  unlex<D>(r, S.np, l);
  const long long rb = rowptr[S.row_off + r], re = rowptr[S.row_off + r + 1];
  for (long long q = rb; q < re; ++q)
    for (int f = 0; f < 3; ++f) val[f * nnz_total + q] = 0.0;
  const double vol = kuhn_volume<D>(L.G.hc);
  for_simplices_at<D>(l, S.nc, [&](const int c[3], int t, int i) {
    double G[D + 1][D];
    kuhn_grad<D>(c_kt[D].perm[t], L.G.hc, G);
    double GG[D + 1][D + 1];
    for (int k = 0; k <= D; ++k)
      for (int m = 0; m <= D; ++m) {
        double s = 0.0;
        for (int a = 0; a < D; ++a) s += G[k][a] * G[m][a];
        GG[k][m] = s;
      }
    const double se = cell_mult<D>(kmult, L, S, c, nH);
    for (int j = 0; j < N; ++j) {
      int v[3];
      for (int a = 0; a < D; ++a) v[a] = 2 * c[a] + c_kt[D].off[t][j][a];
      const int cj = (int)lex<D>(v, S.np);
      double kij = 0.0;
      for (int k = 0; k <= D; ++k)
        for (int m = 0; m <= D; ++m) kij += ref->G22[i][k][j][m] * GG[k][m];
      const double mij = vol * ref->M22[i][j];
      kij *= vol;
      const long long q = find_slot(col, rb, re, cj);
      for (int f = 0; f < 3; ++f) val[f * nnz_total + q] += (pc.c[f] + se * pc.gamma[f]) * mij + se * pc.kappa[f] * kij;
    }
  });
  const long long qd = find_slot(col, rb, re, r);
  for (int f = 0; f < 3; ++f) diag[f * rows_total + S.row_off + r] = val[f * nnz_total + qd];
}

// isq = 1/sqrt(diag) on free rows, 0 on fixed rows (Dirichlet dir / artificial, C4, C5)
template <int D>
__global__ void k_porous_isq(const SysDesc* __restrict__ sys, Level L, const double* __restrict__ diag,
                             double* __restrict__ isq, long long rows_total) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  int l[3] = {0, 0, 0};
  unlex<D>(r, S.np, l);
  const bool fixed = node_class<D>(L.G, S, l) >= CL_ART;
  for (int f = 0; f < 3; ++f) {
    const long long k = f * rows_total + S.row_off + r;
    isq[k] = fixed ? 0.0 : 1.0 / sqrt(diag[k]);
  }
}

// symmetric Jacobi scaling  A~ = D^-1/2 A D^-1/2  (fixed rows and columns become zero)
template <int D>
__global__ void k_porous_scale(const SysDesc* __restrict__ sys, const long long* __restrict__ rowptr,
                               const int* __restrict__ col, double* __restrict__ val, long long nnz_total,
                               const double* __restrict__ isq, long long rows_total) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  const long long rb = rowptr[S.row_off + r], re = rowptr[S.row_off + r + 1];
  for (int f = 0; f < 3; ++f) {
    const double* is = isq + f * rows_total + S.row_off;
    const double ir = is[r];
    for (long long q = rb; q < re; ++q) val[f * nnz_total + q] *= ir * is[col[q]];
  }
}

// ---------------------------------------------------------------------------------------------
// prolongation: evaluate a coarse P2 / P1 finite-element function of the whole region at a fine
// half-grid point g (exact, nested meshes P:443-444).  Weights are exact rationals over 2 R^2,
// computed from integer numerators and rounded once.
template <int D>
__device__ double prolong_p2(const double* __restrict__ uc, const int nH[3], int R, const int g[3]) {
  int cell[3], num[3], ord[3] = {0, 1, 2};
  for (int a = 0; a < D; ++a) {
    cell[a] = min(g[a] / (2 * R), nH[a] - 1);
    num[a] = g[a] - 2 * R * cell[a];
  }
  for (int a = 1; a < D; ++a)  // stable sort of axes by num, descending
    for (int b = a; b > 0 && num[ord[b]] > num[ord[b - 1]]; --b) {
      int tmp = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = tmp;
    }
  long long lam[4];
  lam[0] = 2 * R - num[ord[0]];
  for (int k = 1; k < D; ++k) lam[k] = num[ord[k - 1]] - num[ord[k]];
  lam[D] = num[ord[D - 1]];
  int V[4][3];
  for (int a = 0; a < D; ++a) V[0][a] = 2 * cell[a];
  for (int k = 1; k <= D; ++k) {
    for (int a = 0; a < D; ++a) V[k][a] = V[k - 1][a];
    V[k][ord[k - 1]] += 2;
  }
  int shp[3] = {2 * nH[0] + 1, 2 * nH[1] + 1, 2 * nH[2] + 1};
  const double den = 2.0 * (double)R * (double)R;
  double s = 0.0;
  for (int k = 0; k <= D; ++k) {
    const long long w = lam[k] * (lam[k] - R);  // lam (2 lam - 1) = n (n - R) / (2 R^2)
    if (w != 0) s += ((double)w / den) * uc[lex<D>(V[k], shp)];
  }
  for (int a = 0; a <= D; ++a)
    for (int b = a + 1; b <= D; ++b) {
      const long long w = 2 * lam[a] * lam[b];  // 4 lam_a lam_b = 2 n_a n_b / (2 R^2)
      if (w != 0) {
        int E[3];
        for (int c = 0; c < D; ++c) E[c] = (V[a][c] + V[b][c]) / 2;
        s += ((double)w / den) * uc[lex<D>(E, shp)];
      }
    }
  return s;
}

template <int D>
__device__ double prolong_p1(const double* __restrict__ pc, const int nH[3], int R, const int g[3]) {
  int cell[3], num[3], ord[3] = {0, 1, 2};
  for (int a = 0; a < D; ++a) {
    cell[a] = min(g[a] / (2 * R), nH[a] - 1);
    num[a] = g[a] - 2 * R * cell[a];
  }
  for (int a = 1; a < D; ++a)
    for (int b = a; b > 0 && num[ord[b]] > num[ord[b - 1]]; --b) {
      int tmp = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = tmp;
    }
  long long lam[4];
  lam[0] = 2 * R - num[ord[0]];
  for (int k = 1; k < D; ++k) lam[k] = num[ord[k - 1]] - num[ord[k]];
  lam[D] = num[ord[D - 1]];
  int V[3];
  int shp[3] = {nH[0] + 1, nH[1] + 1, nH[2] + 1};
  for (int a = 0; a < D; ++a) V[a] = cell[a];
  double s = 0.0;
  const double den = 2.0 * (double)R;
  for (int k = 0; k <= D; ++k) {
    if (k > 0) V[ord[k - 1]] += 1;
    if (lam[k] != 0) s += ((double)lam[k] / den) * pc[lex<D>(V, shp)];
  }
  return s;
}

// ---------------------------------------------------------------------------------------------
// porous per-step preparation (one thread per box node), Algorithm 3 Step 3(1) / Step 1:
//   base = P p_iH^{n+1} (fine) or p_iH^n (coarse), z = base with I_h g(t_{n+1}) on dir nodes (C5),
//   lag = lagged field p~^n (mode B composite / mode A P p_H^n + e_j^n / coarse p_H^n),
//   q = forcing at t_{n+1} (C13: loads M I_h q), w = -(u^n . e_last) on Gamma nodes for the flux
//   <u^n . n_c, v_F> (n_c = -e_last).
struct PorousPrepArgs {
  const double* coarse_new[3];   // coarse porous state at n+1 (fine stage) or n (coarse stage)
  const double* coarse_old[3];   // coarse porous state at n
  const double* coarse_u_old;    // conduit velocity at n, last component (for the flux): coarse, or (Algorithm 1
                                 // on T_h) the fine composite
  int nHu[3], Ru;                // cells of that velocity's mesh per axis and fine cells per cell of it
  const double* comp[3];         // global fine composite (mode B)
  const double* ecorr;           // mode A stored corrections (3 fields, row space) or NULL
  int nHp[3], nHc[3];            // coarse cells of porous / conduit regions
  int Rp;                        // fine cells per coarse cell (1 on the coarse stage)
  int np_glob[3];                // P2 nodes per axis of the global fine porous region
  int conduit_gamma_g;           // conduit half-grid index of Gamma (0)
  int mode;                      // 0 composite (B), 1 subdomain (A), 2 coarse
  int zero_base;                 // 1: base 0, the unknown is the full field (Algorithm 1 on T_h: no cancellation
                                 //    in the right-hand side, so the C19 test is attainable)
  double t;                      // t_{n+1}
};

template <int D>
__global__ void k_porous_prep(const SysDesc* __restrict__ sys, Level L, ProbData pd, Coef co, PorousPrepArgs A,
                              double* __restrict__ base, double* __restrict__ z, double* __restrict__ lag,
                              double* __restrict__ q, double* __restrict__ wg, long long rows_total) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  int l[3] = {0, 0, 0}, g[3] = {0, 0, 0};
  unlex<D>(r, S.np, l);
  double x[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) {
    g[a] = 2 * S.c0[a] + l[a];
    x[a] = L.G.lo[a] + g[a] * L.G.hg[a];
  }
  const int cls = node_class<D>(L.G, S, l);
  double gval[3], qv[3];
  porous_values<D>(pd, x, A.t, gval);
  porous_forcing<D>(pd, co, x, A.t, qv);
  const long long k0 = S.row_off + r;
  for (int f = 0; f < 3; ++f) {
    const long long k = f * rows_total + k0;
    double b, lg;
    if (A.mode == 2) {
      b = A.zero_base ? 0.0 : A.coarse_new[f][lex<D>(g, A.np_glob)];
      lg = A.coarse_old[f][lex<D>(g, A.np_glob)];
    } else {
      b = prolong_p2<D>(A.coarse_new[f], A.nHp, A.Rp, g);
      if (A.mode == 0) lg = A.comp[f][lex<D>(g, A.np_glob)];
      else lg = prolong_p2<D>(A.coarse_old[f], A.nHp, A.Rp, g) + A.ecorr[k];
    }
    base[k] = b;
    z[k] = cls == CL_DIR ? gval[f] : b;
    lag[k] = lg;
    q[k] = qv[f];
  }
  double w = 0.0;
  if (g[D - 1] == L.G.gamma_g) {
    int gc[3] = {g[0], g[1], g[2]};
    gc[D - 1] = A.conduit_gamma_g;
    w = -prolong_p2<D>(A.coarse_u_old, A.nHu, A.Ru, gc);
  }
  wg[k0] = w;
}

// Facets of Gamma around a node on Gamma: (D-1)-dimensional Kuhn simplices over the tangential axes.
template <int D, class F>
__device__ __forceinline__ void for_facets_at(const int l[3], const int nc[3], F&& f) {
  if (D == 2) {
    int lt[3] = {l[0], 0, 0}, nct[3] = {nc[0], 0, 0};
    for_simplices_at<1>(lt, nct, f);
  } else {
    int lt[3] = {l[0], l[1], 0}, nct[3] = {nc[0], nc[1], 0};
    for_simplices_at<2>(lt, nct, f);
  }
}

// porous right-hand side in correction form, matrix-free:  b~ = isq * (b_load - A z)
//   b_load_F = M (c_F p~_F + q_F) + M[gFf] p~_f + <w, v>_Gamma
//   b_load_f = M (c_f p~_f + q_f) + M[gfm] p~_m + M[gFf] p~_F
//   b_load_m = M (c_m p~_m + q_m) + M[gfm] p~_f            (P:1279-1310 in full-field form)
template <int D>
__global__ void k_porous_rhs(const SysDesc* __restrict__ sys, Level L, PorousCoefs pc,
                             const double* __restrict__ kmult, int nH0, int nH1, int nH2,
                             const RefT<D>* __restrict__ ref, const double* __restrict__ z,
                             const double* __restrict__ lag, const double* __restrict__ q,
                             const double* __restrict__ wg, const double* __restrict__ isq,
                             double* __restrict__ rhs, double* __restrict__ bnorm_w, long long rows_total) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  constexpr int N = n2_of(D);
  const int nH[3] = {nH0, nH1, nH2};
  int l[3] = {0, 0, 0};
  unlex<D>(r, S.np, l);
  const long long o = S.row_off;
  const double* zf[3] = {z + o, z + rows_total + o, z + 2 * rows_total + o};
  const double* lf[3] = {lag + o, lag + rows_total + o, lag + 2 * rows_total + o};
  const double* qf[3] = {q + o, q + rows_total + o, q + 2 * rows_total + o};
  double b[3] = {0, 0, 0};
  const double vol = kuhn_volume<D>(L.G.hc);
  for_simplices_at<D>(l, S.nc, [&](const int c[3], int t, int i) {
    double G[D + 1][D];
    kuhn_grad<D>(c_kt[D].perm[t], L.G.hc, G);
    double GG[D + 1][D + 1];
    for (int k = 0; k <= D; ++k)
      for (int m = 0; m <= D; ++m) {
        double s = 0.0;
        for (int a = 0; a < D; ++a) s += G[k][a] * G[m][a];
        GG[k][m] = s;
      }
    const double se = cell_mult<D>(kmult, L, S, c, nH);
    for (int j = 0; j < N; ++j) {
      int v[3];
      for (int a = 0; a < D; ++a) v[a] = 2 * c[a] + c_kt[D].off[t][j][a];
      const int cj = (int)lex<D>(v, S.np);
      double kij = 0.0;
      for (int k = 0; k <= D; ++k)
        for (int m = 0; m <= D; ++m) kij += ref->G22[i][k][j][m] * GG[k][m];
      kij *= vol;
      const double mij = vol * ref->M22[i][j];
      const double lm = lf[0][cj], lfv = lf[1][cj], lF = lf[2][cj];
      // field 2 = F
      b[2] += mij * (pc.c[2] * lF + qf[2][cj] + se * pc.gFf * lfv);
      b[1] += mij * (pc.c[1] * lfv + qf[1][cj] + se * (pc.gfm * lm + pc.gFf * lF));
      b[0] += mij * (pc.c[0] * lm + qf[0][cj] + se * pc.gfm * lfv);
      for (int f = 0; f < 3; ++f)
        b[f] -= ((pc.c[f] + se * pc.gamma[f]) * mij + se * pc.kappa[f] * kij) * zf[f][cj];
    }
  });
  if (S.has_gamma && 2 * S.c0[D - 1] + l[D - 1] == L.G.gamma_g) {
    double hf[3] = {L.G.hc[0], L.G.hc[1], 0};
    const double fvol = kuhn_volume<D - 1>(hf);
    for_facets_at<D>(l, S.nc, [&](const int c[3], int t, int i) {
      for (int j = 0; j < n2_of(D - 1); ++j) {
        int v[3] = {0, 0, 0};
        for (int a = 0; a < D - 1; ++a) v[a] = 2 * c[a] + c_kt[D - 1].off[t][j][a];
        v[D - 1] = l[D - 1];
        b[2] += fvol * ref->MF[i][j] * wg[o + lex<D>(v, S.np)];
      }
    });
  }
  for (int f = 0; f < 3; ++f) {
    const long long k = f * rows_total + o + r;
    const double is = isq[k];
    rhs[k] = is * b[f];
    // weight 1/isq^2 = diag for the unscaled residual norm (C19)
    bnorm_w[k] = is > 0.0 ? 1.0 / (is * is) : 0.0;
  }
}

// write-back (Algorithm 3 Step 4): full = z + e on owned nodes (C3); mode A keeps e_j.
template <int D>
__device__ __forceinline__ bool owns(const Level& L, const SysDesc& S, const int g[3]) {
  if (S.level == 0) return true;
  for (int a = 0; a < D; ++a) {
    int o = min(g[a] / (2 * L.core[a]), L.m[a] - 1);
    if (o != S.pos[a]) return false;
  }
  return true;
}

template <int D>
__global__ void k_porous_writeback(const SysDesc* __restrict__ sys, Level L, const double* __restrict__ z,
                                   const double* __restrict__ e, const double* __restrict__ isq,
                                   const double* __restrict__ base, double* __restrict__ ecorr, double* out0,
                                   double* out1, double* out2, int np0, int np1, int np2, long long rows_total) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  int l[3] = {0, 0, 0}, g[3] = {0, 0, 0};
  unlex<D>(r, S.np, l);
  for (int a = 0; a < D; ++a) g[a] = 2 * S.c0[a] + l[a];
  const int npg[3] = {np0, np1, np2};
  double* out[3] = {out0, out1, out2};
  const bool own = owns<D>(L, S, g);
  const long long gi = lex<D>(g, npg);
  for (int f = 0; f < 3; ++f) {
    const long long k = f * rows_total + S.row_off + r;
    const double full = z[k] + isq[k] * e[k];  // e solved in the scaled variable
    if (own) out[f][gi] = full;
    if (ecorr) ecorr[k] = full - base[k];
  }
}

}  // namespace lp
