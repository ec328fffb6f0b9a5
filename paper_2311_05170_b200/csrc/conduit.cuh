// conduit.cuh -- Taylor-Hood P2-P1 conduit operators (row-gather, atomic-free).
//
// Fine correction (Algorithm 3 Step 3(2), eq. uclocalFully), full-field form with
// U = P u_cH^{n+1} and u = U + e, p = P p_H^{n+1} + delta:
//   (eta/dt)(u - u~^n, v) + 2 nu eta (D u, D v) + (eta nu alpha/sqrt(k_F)) <P_tau u, P_tau v>_Gamma
//   + eta((u.grad)U, v) + eta((U.grad)u, v) - eta((U.grad)U, v) - eta(p, div v)
//   = eta(f, v) - (eta/rho)<P p_FH^n, v.n_c>_Gamma - (eta nu alpha sqrt(k_F)/mu)<grad_tau P p_FH^n, P_tau v>_Gamma,
//   eta(q, div u) = 0,
// Coarse step (eq. pcFully) by Picard: the same operator without the reaction term
// eta((u.grad)U, v) and without -eta((U.grad)U, v), wind W = previous iterate (C11).
// Signs: n_c = -e_last on Gamma; friction coefficient eta nu alpha sqrt(d)/sqrt(tr Pi) with
// Pi = k_F I; tangential load coefficient eta nu alpha sqrt(k_F)/mu.
#pragma once
#include "assembly.cuh"

namespace lp {

struct ConduitCoefs {
  double eta, nu, alpha, rho, mu, kF, dt;
  double schur_w;  // pressure scaling numerator: nu + h^2/(c dt) (preconditioner only)
  double vel_w;    // velocity scaling factor of the preconditioner levels (1: plain Jacobi)
};

template <int D>
__device__ __forceinline__ double gamma_mult(const double* __restrict__ kmult, const Level& L, const SysDesc& S,
                                             const int c[3], const int nHp[3]) {
  // k_F multiplier of the porous coarse cell under a Gamma facet at tangential box cell c (C15)
  if (!kmult) return 1.0;
  int cc[3];
  for (int a = 0; a < D - 1; ++a) cc[a] = (S.c0[a] + c[a]) / L.G.R;
  cc[D - 1] = nHp[D - 1] - 1;
  return kmult[lex<D>(cc, nHp)];
}

// length of the comp-0 block of a velocity row (first column >= n2)
__device__ __forceinline__ long long block_len(const int* __restrict__ col, long long rb, long long re, int n2) {
  return find_slot(col, rb, re, n2) - rb;
}

// constant part, unscaled: (eta/dt) M + 2 nu eta D:D + friction_Gamma; -eta(p, div v); eta(q, div u)
template <int D>
__global__ void k_conduit_const(const SysDesc* __restrict__ sys, Level L, ConduitCoefs cc,
                                const double* __restrict__ kmult, int nHp0, int nHp1, int nHp2,
                                const RefT<D>* __restrict__ ref, const long long* __restrict__ rowptr,
                                const int* __restrict__ col, double* __restrict__ aconst) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  constexpr int N = n2_of(D);
  const int nHp[3] = {nHp0, nHp1, nHp2};
  const long long rb = rowptr[S.row_off + r], re = rowptr[S.row_off + r + 1];
  for (long long q = rb; q < re; ++q) aconst[q] = 0.0;
  const double vol = kuhn_volume<D>(L.G.hc);
  const int shp1[3] = {S.nc[0] + 1, S.nc[1] + 1, S.nc[2] + 1};
  int l[3] = {0, 0, 0};
  if (r < D * S.n2) {
    const int a = r / S.n2;
    unlex<D>(r % S.n2, S.np, l);
    const long long Ln = block_len(col, rb, re, S.n2);
    for_simplices_at<D>(l, S.nc, [&](const int c[3], int t, int i) {
      double G[D + 1][D];
      kuhn_grad<D>(c_kt[D].perm[t], L.G.hc, G);
      for (int j = 0; j < N; ++j) {
        int v[3];
        for (int e = 0; e < D; ++e) v[e] = 2 * c[e] + c_kt[D].off[t][j][e];
        const int cj = (int)lex<D>(v, S.np);
        const long long p0 = find_slot(col, rb, rb + Ln, cj);
        // S_xy = int d_x phi_i d_y phi_j
        double Sxy[D][D];
        for (int x = 0; x < D; ++x)
          for (int y = 0; y < D; ++y) {
            double s = 0.0;
            for (int k = 0; k <= D; ++k)
              for (int m = 0; m <= D; ++m) s += ref->G22[i][k][j][m] * G[k][x] * G[m][y];
            Sxy[x][y] = vol * s;
          }
        double lap = 0.0;
        for (int x = 0; x < D; ++x) lap += Sxy[x][x];
        const double nue = cc.nu * cc.eta;
        for (int b = 0; b < D; ++b) {
          double v_ab = nue * ((a == b ? lap : 0.0) + Sxy[b][a]);
          if (a == b) v_ab += (cc.eta / cc.dt) * vol * ref->M22[i][j];
          aconst[p0 + b * Ln] += v_ab;
        }
      }
      // pressure columns: -eta int psi_m d_a phi_i
      for (int m = 0; m <= D; ++m) {
        int v[3];
        for (int e = 0; e < D; ++e) v[e] = (2 * c[e] + c_kt[D].off[t][m][e]) >> 1;
        const int key = D * S.n2 + (int)lex<D>(v, shp1);
        double s = 0.0;
        for (int k = 0; k <= D; ++k) s += ref->D12[m][i][k] * G[k][a];
        aconst[find_slot(col, rb + D * Ln, re, key)] += -cc.eta * vol * s;
      }
    });
    // Gamma friction on tangential components
    if (a < D - 1 && S.has_gamma && 2 * S.c0[D - 1] + l[D - 1] == L.G.gamma_g) {
      double hf[3] = {L.G.hc[0], L.G.hc[1], 0};
      const double fvol = kuhn_volume<D - 1>(hf);
      for_facets_at<D>(l, S.nc, [&](const int c[3], int t, int i) {
        const double kF = cc.kF * gamma_mult<D>(kmult, L, S, c, nHp);
        const double fric = cc.eta * cc.nu * cc.alpha / sqrt(kF);
        for (int j = 0; j < n2_of(D - 1); ++j) {
          int v[3] = {0, 0, 0};
          for (int e = 0; e < D - 1; ++e) v[e] = 2 * c[e] + c_kt[D - 1].off[t][j][e];
          v[D - 1] = l[D - 1];
          const int cj = (int)lex<D>(v, S.np);
          aconst[find_slot(col, rb, rb + Ln, cj) + a * Ln] += fric * fvol * ref->MF[i][j];
        }
      });
    }
  } else {
    // continuity row of vertex k: eta int psi_k d_b phi_j
    unlex<D>(r - D * S.n2, shp1, l);
    for (int e = 0; e < D; ++e) l[e] *= 2;
    const long long Ln = (re - rb) / D;
    for_simplices_at<D>(l, S.nc, [&](const int c[3], int t, int i) {
      double G[D + 1][D];
      kuhn_grad<D>(c_kt[D].perm[t], L.G.hc, G);
      for (int j = 0; j < N; ++j) {
        int v[3];
        for (int e = 0; e < D; ++e) v[e] = 2 * c[e] + c_kt[D].off[t][j][e];
        const int cj = (int)lex<D>(v, S.np);
        const long long p0 = find_slot(col, rb, rb + Ln, cj);
        for (int b = 0; b < D; ++b) {
          double s = 0.0;
          for (int k = 0; k <= D; ++k) s += ref->D12[i][j][k] * G[k][b];
          aconst[p0 + b * Ln] += cc.eta * vol * s;
        }
      }
    });
  }
}

// right preconditioner (diagonal): velocity 1/diag(A_const); pressure schur_w/(eta int psi_k);
// zero on fixed rows (velocity dir/art nodes, pressure vertices on artificial faces, C4).
template <int D>
__global__ void k_conduit_scale(const SysDesc* __restrict__ sys, Level L, ConduitCoefs cc,
                                const long long* __restrict__ rowptr, const int* __restrict__ col,
                                const double* __restrict__ aconst, double* __restrict__ s) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  const long long rb = rowptr[S.row_off + r], re = rowptr[S.row_off + r + 1];
  int l[3] = {0, 0, 0};
  double v;
  if (r < D * S.n2) {
    unlex<D>(r % S.n2, S.np, l);
    const bool fixed = node_class<D>(L.G, S, l) >= CL_ART;
    v = fixed ? 0.0 : cc.vel_w / aconst[find_slot(col, rb, re, r)];
  } else {
    const int shp1[3] = {S.nc[0] + 1, S.nc[1] + 1, S.nc[2] + 1};
    unlex<D>(r - D * S.n2, shp1, l);
    for (int e = 0; e < D; ++e) l[e] *= 2;
    double mk = 0.0;
    const double vol = kuhn_volume<D>(L.G.hc);
    for_simplices_at<D>(l, S.nc, [&](const int*, int, int) { mk += vol / (D + 1); });
    v = vertex_on_art<D>(S, l) ? 0.0 : cc.schur_w / (cc.eta * mk);
  }
  s[S.row_off + r] = v;
}

// per-step preparation (one thread per P2 node or P1 vertex)
struct ConduitPrepArgs {
  const double* cu_new;   // coarse conduit velocity (D comps, coarse P2 layout) at n+1 (fine) / Picard iterate (coarse)
  const double* cp_new;   // coarse conduit pressure at n+1 (fine) / Picard iterate (coarse)
  const double* cu_old;   // coarse conduit velocity at n
  const double* cpF_old;  // coarse porous p_F at n
  const double* comp_u;   // global fine composite velocity (mode B)
  const double* ecorr;    // mode A corrections (row space) or NULL
  int nHc[3], nHp[3];
  int R;
  int np_glob[3];         // P2 nodes per axis of the level's conduit region
  long long n2_glob;      // P2 nodes of the level's conduit region (component stride)
  int porous_gamma_g;     // half-grid index of Gamma in the porous region at the coarse level x R
  int mode;               // 0 fine composite (B), 1 fine subdomain (A), 2 coarse Picard, 3 operator only (U)
  int zero_base;          // 1: base 0 (the unknown is the full field), wind = cu_new (Algorithm 1 on T_h)
  double t;
};

template <int D>
__global__ void k_conduit_prep(const SysDesc* __restrict__ sys, Level L, ProbData pd, Coef co, ConduitPrepArgs A,
                               double* __restrict__ base, double* __restrict__ z, double* __restrict__ W,
                               double* __restrict__ lag, double* __restrict__ f, double* __restrict__ pfg) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.n2 + S.n1) return;
  const long long o = S.row_off;
  int l[3] = {0, 0, 0}, g[3] = {0, 0, 0};
  double x[3] = {0, 0, 0};
  if (r < S.n2) {
    unlex<D>(r, S.np, l);
    for (int a = 0; a < D; ++a) {
      g[a] = 2 * S.c0[a] + l[a];
      x[a] = L.G.lo[a] + g[a] * L.G.hg[a];
    }
    const int cls = node_class<D>(L.G, S, l);
    const bool top = g[D - 1] == 2 * L.G.n[D - 1];
    double gv[3], fv[3];
    velocity_values<D>(pd, x, A.t, top, gv);
    velocity_forcing<D>(pd, co, x, A.t, fv);
    const int shpH[3] = {2 * A.nHc[0] + 1, 2 * A.nHc[1] + 1, 2 * A.nHc[2] + 1};
    const long long n2H = (long long)shpH[0] * shpH[1] * (D > 2 ? shpH[2] : 1);
    for (int a = 0; a < D; ++a) {
      const long long k = o + a * S.n2 + r;
      double b, lg;
      if (A.mode == 3) {
        b = prolong_p2<D>(A.cu_new + a * n2H, A.nHc, A.R, g);
        base[k] = b;
        W[k] = b;
        z[k] = b;
        lag[k] = 0.0;
        f[k] = 0.0;
        continue;
      }
      if (A.mode == 2) {
        const long long gi = lex<D>(g, A.np_glob);
        b = A.cu_new[a * A.n2_glob + gi];
        lg = A.cu_old[a * A.n2_glob + gi];
      } else {
        b = prolong_p2<D>(A.cu_new + a * n2H, A.nHc, A.R, g);
        if (A.mode == 0) lg = A.comp_u[a * A.n2_glob + lex<D>(g, A.np_glob)];
        else lg = prolong_p2<D>(A.cu_old + a * n2H, A.nHc, A.R, g) + A.ecorr[k];
      }
      W[k] = b;
      if (A.zero_base) b = 0.0;
      base[k] = b;
      z[k] = cls == CL_DIR ? gv[a] : b;
      lag[k] = lg;
      f[k] = fv[a];
    }
    double pf = 0.0;
    if (A.mode != 3 && g[D - 1] == L.G.gamma_g) {
      int gp[3] = {g[0], g[1], g[2]};
      gp[D - 1] = A.porous_gamma_g;
      pf = prolong_p2<D>(A.cpF_old, A.nHp, A.R, gp);
    }
    pfg[o + r] = pf;
  } else {
    const int k1 = r - S.n2;
    const int shp1[3] = {S.nc[0] + 1, S.nc[1] + 1, S.nc[2] + 1};
    unlex<D>(k1, shp1, l);
    for (int a = 0; a < D; ++a) g[a] = 2 * (S.c0[a] + l[a]);
    double b;
    if (A.mode == 3) {
      b = 0.0;
    } else if (A.mode == 2) {
      int v[3];
      for (int a = 0; a < D; ++a) v[a] = g[a] / 2;
      const int shpg1[3] = {(A.np_glob[0] + 1) / 2, (A.np_glob[1] + 1) / 2, (A.np_glob[2] + 1) / 2};
      b = A.cp_new[lex<D>(v, shpg1)];
    } else {
      b = prolong_p1<D>(A.cp_new, A.nHc, A.R, g);
    }
    const long long k = o + D * S.n2 + k1;
    if (A.zero_base) b = 0.0;
    base[k] = b;
    z[k] = b;
  }
}

// Per-step operator, one WARP per velocity P2 node (all D rows of the node) or per continuity row.  Everything the
// element walk touches is staged in shared memory first, with independent coalesced loads: the node's rows of
// aconst, its column list, and the wind W and the load (eta f + (eta/dt) u~^n) at its P2 neighbours -- the nodes of
// all simplices around it.  Every simplex then adds its convection / Newton-reaction block in one conflict-free
// round (lane = (j, b): element node j, column block b; distinct lanes hit distinct entries; the position of node j
// in the row by binary search in the staged column list), and the finished rows are masked, scaled and written once
// (coalesced): one read of aconst, one write of aout, no global access inside the walk.  Barycentric gradients of
// Kuhn simplices are +-1/h per axis: sum_k C3[..][k] G[k][c] = (C3[..][p + 1] - C3[..][p]) / h_c with p the rank of
// axis c in the simplex's permutation (C3 in shared memory).
//   A' = mask * (A_const + eta N(W) [+ eta R(U)]) * diag(s)
//   rhs = mask * (b_load - A z), b_load = eta M f + (eta/dt) M u~^n [+ eta N(U) U] + Gamma loads.
template <int D>
struct CStepW;
template <int D>
constexpr int cstep_rel_bytes() {  // relative offset codes rel[t][i][m] (nt x N x N bytes), padded to 16 B
  return (nt_of(D) * n2_of(D) * n2_of(D) + 15) & ~15;
}
template <int D>
constexpr int cstep_cl_bytes() {  // simplex lists per parity class: (1 << D) x 8 nt shorts, then (1 << D) counts
  return (((1 << D) * 8 * nt_of(D) * 2 + (1 << D) * 4) + 15) & ~15;
}
template <int D>
constexpr int cstep_tab_bytes() {  // DA, DB (D x N^3 each), M22 (N^2), rel codes, simplex lists: 16-byte multiple
  return (int)sizeof(double) * (2 * D * n2_of(D) * n2_of(D) * n2_of(D) + n2_of(D) * n2_of(D)) + cstep_rel_bytes<D>() +
         cstep_cl_bytes<D>();
}
template <int D, int WPB>
constexpr size_t cstep_smem() {  // the tables, then one CStepW per warp
  return cstep_tab_bytes<D>() + WPB * sizeof(CStepW<D>);
}
template <int D>
struct CStepW {
  static constexpr int N = n2_of(D);
  static constexpr int RMAX = D == 3 ? 232 : 56;  // >= longest velocity row (checked at setup): 3 x 65 + 27 / 2 x 19 + 9
  static constexpr int LMAX = D == 3 ? 72 : 24;   // >= P2 neighbours of a node
  double row[D][RMAX];  // the node's D rows
  double Uw[D][LMAX];   // wind at the P2 neighbours (row order)
  double Lw[D][LMAX];   // eta f + (eta/dt) u~^n at the P2 neighbours
  int colr[RMAX];       // column list of the rows (block 0: P2 neighbours, ascending)
  int slot[N];          // position of the current simplex's nodes in the neighbour list
  double Ue[D * N];     // wind at the current simplex's nodes, component-major (Ue[a N + m])
  unsigned char map[D == 3 ? 128 : 32];  // slot of the P2 neighbour at half-grid offset d in [-2, 2]^D (code
                                         // sum_a (d_a + 2) 5^a)
};


// the reference tables of k_conduit_step_w (one CTA, once per context): built in shared memory with the kernel's
// layout, then stored to tab (cstep_tab_bytes<D>() bytes) for the per-CTA copies
template <int D>
__global__ void k_cstep_tables(const RefT<D>* __restrict__ ref, double* __restrict__ tab) {
  constexpr int N = n2_of(D);
  constexpr int NT3 = D * N * N * N;
  extern __shared__ __align__(16) double cstep_dyn[];
  double* DA = cstep_dyn;
  double* DB = cstep_dyn + NT3;
  double* sM = cstep_dyn + 2 * NT3;
  unsigned char* rel = reinterpret_cast<unsigned char*>(cstep_dyn + 2 * NT3 + N * N);
  short(*s_cl)[8 * nt_of(D)] = reinterpret_cast<short(*)[8 * nt_of(D)]>(rel + cstep_rel_bytes<D>());
  int* s_ncl = reinterpret_cast<int*>(rel + cstep_rel_bytes<D>() + (1 << D) * 8 * nt_of(D) * 2);
  for (int k = threadIdx.x; k < NT3; k += blockDim.x) {
    const int j = k % N, m = (k / N) % N, i = (k / (N * N)) % N, p = k / (N * N * N);
    DA[k] = ref->C3[i][m][j][p + 1] - ref->C3[i][m][j][p];
    DB[k] = ref->C3[i][j][m][p + 1] - ref->C3[i][j][m][p];
  }
  for (int k = threadIdx.x; k < N * N; k += blockDim.x) sM[k] = (&ref->M22[0][0])[k];
  // simplex lists per parity class of a node (for_simplices_at's enumeration with the cube candidates of an interior
  // node: per even axis the cubes l/2 - 1 and l/2, per odd axis (l - 1)/2)
    if (threadIdx.x < (1 << D)) {
    const int pcl = threadIdx.x;
    int n = 0;
    const int n2 = D > 2 ? ((pcl >> 2) & 1 ? 1 : 2) : 1, n1 = D > 1 ? ((pcl >> 1) & 1 ? 1 : 2) : 1;
    const int n0 = (pcl & 1) ? 1 : 2;
    for (int i2 = 0; i2 < n2; ++i2)
      for (int i1 = 0; i1 < n1; ++i1)
        for (int i0 = 0; i0 < n0; ++i0) {
          const int ii[3] = {i0, i1, i2};
          int code = 0, f = 1, dcm = 0;
          for (int a = 0; a < D; ++a, f *= 3) {
            int o;  // offset of the node in the cube (half-grid units)
            if ((pcl >> a) & 1) {
              o = 1;
            } else if (ii[a] == 0) {
              o = 2;  // cube l/2 - 1
              dcm |= 1 << a;
            } else {
              o = 0;  // cube l/2
            }
            code += o * f;
          }
          for (int t = 0; t < nt_of(D); ++t) {
            const int i = c_kt[D].lookup[t][code];
            if (i >= 0) s_cl[pcl][n++] = (short)(dcm | (t << 3) | (i << 6));
          }
        }
    s_ncl[pcl] = n;
  }
  for (int k = threadIdx.x; k < nt_of(D) * N * N; k += blockDim.x) {
    const int m = k % N, i = (k / N) % N, t = k / (N * N);
    int code = 0;
    for (int a = 0, f = 1; a < D; ++a, f *= 5) code += (c_kt[D].off[t][m][a] - c_kt[D].off[t][i][a] + 2) * f;
    rel[k] = (unsigned char)code;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < cstep_tab_bytes<D>() / 8; k += blockDim.x) tab[k] = cstep_dyn[k];
}

template <int D, int WPB>
__global__ void __launch_bounds__(WPB * 32)
k_conduit_step_w(const SysDesc* __restrict__ sys, Level L, ConduitCoefs cc, int newton,
                 const double* __restrict__ kmult, int nHp0, int nHp1, int nHp2, const RefT<D>* __restrict__ ref,
                 const long long* __restrict__ rowptr, const int* __restrict__ col,
                 const double* __restrict__ aconst, const double* __restrict__ s, const double* __restrict__ z,
                 const double* __restrict__ W, const double* __restrict__ lag, const double* __restrict__ f,
                 const double* __restrict__ pfg, double* __restrict__ aout, double* __restrict__ rhs, int nbx,
                 int nsys, int* __restrict__ ticket, const double* __restrict__ tab) {
  constexpr int N = n2_of(D);
  constexpr int NT3 = D * N * N * N;
  // barycentric-gradient differences of C3 (gradients of Kuhn simplices are +-1/h: sum_k C3[..][k] G[k][c] =
  // (C3[..][p + 1] - C3[..][p]) / h_c, p = rank of axis c in the simplex's permutation), element node j fastest so
  // that the lanes (j, .) of a warp read consecutive words:
  //   DA[p][i][m][j] = C3[i][m][j][p+1] - C3[i][m][j][p]   (convection: phi_i phi_m d_c phi_j)
  //   DB[p][i][m][j] = C3[i][j][m][p+1] - C3[i][j][m][p]   (reaction:   phi_i phi_j d_c phi_m)
  extern __shared__ __align__(16) double cstep_dyn[];  // DA, DB, M22, rel, then one CStepW per warp (cstep_smem)
  double* DA = cstep_dyn;
  double* DB = cstep_dyn + NT3;
  double* sM = cstep_dyn + 2 * NT3;
  // rel[t][i][m]: offset code of element node m relative to element node i in a simplex of type t (the same for
  // every simplex of that type), so the slot of m in the neighbour list of the row node i is map[rel[t][i][m]]
  unsigned char* rel = reinterpret_cast<unsigned char*>(cstep_dyn + 2 * NT3 + N * N);
  const short(*s_cl)[8 * nt_of(D)] = reinterpret_cast<const short(*)[8 * nt_of(D)]>(rel + cstep_rel_bytes<D>());
  const int* s_ncl = reinterpret_cast<const int*>(rel + cstep_rel_bytes<D>() + (1 << D) * 8 * nt_of(D) * 2);
  CStepW<D>* wb = reinterpret_cast<CStepW<D>*>(reinterpret_cast<unsigned char*>(cstep_dyn) + cstep_tab_bytes<D>());
  // persistent CTAs: the tables are built once per CTA, then the CTA walks blocks of WPB nodes (one warp per node)
  // of the virtual grid (nbx node blocks x nsys systems) with a stride of gridDim.x, or, with a ticket counter
  // (zeroed before the launch), takes the next block in order (the blocks in flight then stay a compact window of
  // the node order: cfg4 DRAM reads 33 -> 15 GB per launch, but the block barrier per step made it slower, 51.7 ->
  // 57.0 ms; the fine family uses the stride).  A grid of one CTA per block makes it the plain one-shot kernel.
  __shared__ int s_next;
  auto grab = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) s_next = (int)gridDim.x + atomicAdd(ticket, 1);
    __syncthreads();
    return s_next;
  };
  if ((long long)gridDim.x >= (long long)nbx * nsys) {  // one CTA per block: an empty block exits before the copy
    const SysDesc S0 = sys[blockIdx.x / nbx];
    if ((int)(blockIdx.x % nbx) * WPB >= S0.n2 + S0.n1) return;
  }
  {  // the tables (built once by k_cstep_tables), copied with 16-byte loads
    const int4* src = reinterpret_cast<const int4*>(tab);
    int4* dst = reinterpret_cast<int4*>(cstep_dyn);
    for (int k = threadIdx.x; k < cstep_tab_bytes<D>() / 16; k += blockDim.x) dst[k] = __ldg(src + k);
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int vb = blockIdx.x; vb < nbx * nsys; vb = ticket ? grab() : vb + (int)gridDim.x) {
  const SysDesc S = sys[vb / nbx];
  const int nitems = S.n2 + S.n1;
  const int r = (vb % nbx) * WPB + w;
  if (r >= nitems) continue;
  __syncwarp();
  const long long o = S.row_off;
  const double* zs = z + o;
  const double* ss = s + o;
  if (r >= S.n2) {  // continuity row: constant (eta (q, div u)), masked and scaled
    const long long row = o + D * S.n2 + (r - S.n2);
    const long long rb = rowptr[row], re = rowptr[row + 1];
    const bool fixed = ss[D * S.n2 + (r - S.n2)] == 0.0;
    double b = 0.0;
    for (long long q = rb + lane; q < re; q += 32) {
      const double v = aconst[q];
      const int cq = col[q];
      b -= v * zs[cq];
      aout[q] = fixed ? 0.0 : v * ss[cq];
    }
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) b += __shfl_xor_sync(0xffffffffu, b, k);
    if (lane == 0) rhs[row] = fixed ? 0.0 : b;
    continue;
  }
  CStepW<D>& B = wb[w];
  const int nHp[3] = {nHp0, nHp1, nHp2};
  int l[3] = {0, 0, 0};
  unlex<D>(r, S.np, l);
  long long rb[D];
#pragma unroll
  for (int a = 0; a < D; ++a) rb[a] = rowptr[o + a * S.n2 + r];
  const int RL = (int)(rowptr[o + r + 1] - rb[0]);  // the D rows of a node have the same length and columns
  const double* Ws = W + o;
  const double* Ls = lag + o;
  const double* Fs = f + o;
  // stage: columns, rows of aconst, wind and loads at the P2 neighbours (independent loads, one latency)
  for (int q = lane; q < RL; q += 32) B.colr[q] = col[rb[0] + q];
#pragma unroll
  for (int a = 0; a < D; ++a)
    for (int q = lane; q < RL; q += 32) B.row[a][q] = aconst[rb[a] + q];
  __syncwarp();
  int Ln = 0;  // P2 neighbours: columns < n2 (ascending), ballot over the staged list
  for (int q0 = 0; q0 < RL; q0 += 32) {
    const bool in = q0 + lane < RL && B.colr[q0 + lane] < S.n2;
    Ln += __popc(__ballot_sync(0xffffffffu, in));
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
    for (int q = lane; q < Ln; q += 32) {
      const int cq = B.colr[q];
      B.Uw[a][q] = Ws[a * S.n2 + cq];
      B.Lw[a][q] = cc.eta * Fs[a * S.n2 + cq] + (cc.eta / cc.dt) * Ls[a * S.n2 + cq];
    }
  // slot map of the P2 neighbours (every element node of a simplex at the node is one of them)
  for (int q = lane; q < Ln; q += 32) {
    int v[3] = {0, 0, 0};
    unlex<D>(B.colr[q], S.np, v);
    int code = 0;
    for (int a = 0, f = 1; a < D; ++a, f *= 5) code += (v[a] - l[a] + 2) * f;
    B.map[code] = (unsigned char)q;
  }
  const double vol = kuhn_volume<D>(L.G.hc);
  const double ev = cc.eta * vol;
  // lane (j, bb): element node j, column block bb (also the component whose right-hand side it accumulates)
  const int jl = lane / D, bl = lane % D;
  const double ihb = 1.0 / L.G.hc[bl], scb = ev / L.G.hc[bl];  // per lane, once
  const bool act = lane < N * D;
  double bpart = 0.0;
  __syncwarp();
  auto simplex = [&](int t, int i) {
    // lane k < D N: slot of element node m = k mod N and the wind component k / N there (one gather per lane;
    // afterwards every lane reads the element's wind at fixed offsets, a broadcast)
    if (act) {
      const int m = lane % N;
      const int sm = B.map[rel[(t * N + i) * N + m]];
      if (lane < N) B.slot[m] = sm;
      B.Ue[lane] = B.Uw[lane / N][sm];
    }
    __syncwarp();
    // lane (j, e): se_e(j) = sum_m W_e(m) DA[p_e][i][m][j] / h_e; cv(j) = eta |K| sum_e se_e(j) (the D lanes of node j
    // exchange their terms, fixed order); the reaction of column block e from DB[p_e]
    const int j = act ? jl : 0;
    const int p = c_kt[D].pos[t][bl];
    const double* da = DA + ((p * N + i) * N) * N + j;
    const double* db = DB + ((p * N + i) * N) * N + j;
    double se = 0.0;
    if (act) {
      const double* ub = B.Ue + bl * N;
#pragma unroll
      for (int m = 0; m < N; ++m) se += ub[m] * da[m * N];
      se *= ihb;
    }
    double cv = 0.0;
#pragma unroll
    for (int e = 0; e < D; ++e) cv += __shfl_sync(0xffffffffu, se, jl * D + e);
    if (act) {
      cv *= ev;
      const int p0 = B.slot[j];
      double self = cv;  // entry (row bl, block bl)
      if (newton) {
        // reaction eta int phi_i phi_j d_bl U_a -> entry (row a, block bl)
        double tv[N];
#pragma unroll
        for (int m = 0; m < N; ++m) tv[m] = db[m * N];
        const double sc = scb;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double rv = 0.0;
          const double* ua = B.Ue + a * N;
#pragma unroll
          for (int m = 0; m < N; ++m) rv += ua[m] * tv[m];
          if (a == bl) self += sc * rv;
          else B.row[a][p0 + bl * Ln] += sc * rv;
        }
        bpart += cv * B.Uw[bl][p0];  // eta ((U.grad)U, v), component bl
      }
      B.row[bl][p0 + bl * Ln] += self;
      bpart += vol * sM[i * N + j] * B.Lw[bl][p0];
    }
    __syncwarp();
  };
  // the simplices at the node, in for_simplices_at's order, from the list of its parity class: entry = (cube
  // offsets dc_a in {-1, 0} of the even axes (bit a set: -1), type t, local index i); a cube outside the box is
  // skipped (uniform across the warp)
  {
    const int pcl = parity_class<D>(l);
    const int ne = s_ncl[pcl];
    for (int e = 0; e < ne; ++e) {
      const int code = s_cl[pcl][e];
      bool ok = true;
#pragma unroll
      for (int a = 0; a < D; ++a)
        if (!(l[a] & 1)) {
          const int ca = (l[a] >> 1) - ((code >> a) & 1);
          ok = ok && ca >= 0 && ca < S.nc[a];
        }
      if (ok) simplex((code >> 3) & 7, code >> 6);
    }
  }
  // right-hand side per component: lanes with bl == a hold its partial sums (fixed-order shuffle tree)
  double bsum[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double v = (act && bl == a) ? bpart : 0.0;
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) v += __shfl_xor_sync(0xffffffffu, v, k);
    bsum[a] = v;
  }
  if (S.has_gamma && 2 * S.c0[D - 1] + l[D - 1] == L.G.gamma_g && lane == 0) {
    double hf[3] = {L.G.hc[0], L.G.hc[1], 0};
    const double fvol = kuhn_volume<D - 1>(hf);
    const double* P = pfg + o;
    for_facets_at<D>(l, S.nc, [&](const int c[3], int t, int i) {
      const double kF = cc.kF * gamma_mult<D>(kmult, L, S, c, nHp);
      const double ctg = cc.eta * cc.nu * cc.alpha * sqrt(kF) / cc.mu;
      double Gt[D][D - 1];
      double hf2[3] = {L.G.hc[0], L.G.hc[1], 0};
      kuhn_grad<D - 1>(c_kt[D - 1].perm[t], hf2, Gt);
      for (int j = 0; j < n2_of(D - 1); ++j) {
        int v[3] = {0, 0, 0};
        for (int e = 0; e < D - 1; ++e) v[e] = 2 * c[e] + c_kt[D - 1].off[t][j][e];
        v[D - 1] = l[D - 1];
        const double pj = P[lex<D>(v, S.np)];
        bsum[D - 1] += (cc.eta / cc.rho) * fvol * ref->MF[i][j] * pj;  // -(eta/rho)<p_F, v.n_c>, n_c = -e_last
        for (int a = 0; a < D - 1; ++a) {
          double tg = 0.0;
          for (int k = 0; k < D; ++k) tg += ref->TF[i][j][k] * Gt[k][a];
          bsum[a] -= ctg * fvol * tg * pj;  // -(eta nu alpha sqrt(k_F)/mu)<grad_tau p_F, P_tau v>
        }
      }
    });
  }
  __syncwarp();
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const bool fixed = ss[a * S.n2 + r] == 0.0;
    double bz = 0.0;
    for (int q = lane; q < RL; q += 32) {
      const double v = B.row[a][q];
      const int cq = B.colr[q];  // the same columns in all D rows of the node
      bz += v * zs[cq];
      aout[rb[a] + q] = fixed ? 0.0 : v * ss[cq];
    }
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) bz += __shfl_xor_sync(0xffffffffu, bz, k);
    if (lane == 0) rhs[o + a * S.n2 + r] = fixed ? 0.0 : bsum[a] - bz;
  }
  }  // virtual blocks
}

// ---- node-blocked copy of a conduit family's CSR operator (krylov.cuh NBMat); item g = item_off + k of system s
// item lengths: node (L, L1) from its comp-0 row, vertex (L, 0) with L = row length / D; counts of columns and values
template <int D>
__global__ void k_nb_len(const SysDesc* __restrict__ sys, const long long* __restrict__ item_off,
                         const long long* __restrict__ rowptr, const int* __restrict__ col, int2* __restrict__ len,
                         long long* __restrict__ ccnt, long long* __restrict__ vcnt) {
  const SysDesc S = sys[blockIdx.y];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= S.n2 + S.n1) return;
  const long long g = item_off[blockIdx.y] + k;
  if (k < S.n2) {
    const long long rb = rowptr[S.row_off + k], re = rowptr[S.row_off + k + 1];
    const int L = (int)block_len(col, rb, re, S.n2);
    const int L1 = (int)(re - rb) - D * L;
    len[g] = make_int2(L, L1);
    ccnt[g] = L + L1;
    vcnt[g] = (long long)D * (re - rb);
  } else {
    const long long row = S.row_off + D * S.n2 + (k - S.n2);
    const long long rb = rowptr[row], re = rowptr[row + 1];
    const int L = (int)((re - rb) / D);
    len[g] = make_int2(L, 0);
    ccnt[g] = L;
    vcnt[g] = re - rb;
  }
}

template <int D>
__global__ void k_nb_cols(const SysDesc* __restrict__ sys, const long long* __restrict__ item_off,
                          const long long* __restrict__ rowptr, const int* __restrict__ col,
                          const int2* __restrict__ len, const long long* __restrict__ cptr, int* __restrict__ nbcol) {
  const SysDesc S = sys[blockIdx.y];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= S.n2 + S.n1) return;
  const long long g = item_off[blockIdx.y] + k;
  const int2 ln = len[g];
  int* out = nbcol + cptr[g];
  const long long row = k < S.n2 ? S.row_off + k : S.row_off + D * S.n2 + (k - S.n2);
  const long long rb = rowptr[row];
  for (int q = 0; q < ln.x; ++q) out[q] = col[rb + q];                                   // P2 nodes (< n2)
  for (int q = 0; q < ln.y; ++q) out[ln.x + q] = col[rb + D * ln.x + q] - D * S.n2;      // P1 vertices
}

// 16-bit column offsets of the node-blocked operator: per item the bases (first P2 column, first P1 column; the
// blocks are sorted ascending) and column - base; *bad set when an offset does not fit 16 bits
template <int D>
__global__ void k_nb_cols16(const SysDesc* __restrict__ sys, const long long* __restrict__ item_off,
                            const int2* __restrict__ len, const long long* __restrict__ cptr,
                            const int* __restrict__ nbcol, unsigned short* __restrict__ col16,
                            int2* __restrict__ cbase, int* __restrict__ bad) {
  const SysDesc S = sys[blockIdx.y];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= S.n2 + S.n1) return;
  const long long g = item_off[blockIdx.y] + k;
  const int2 ln = len[g];
  const int* in = nbcol + cptr[g];
  const int b2 = ln.x > 0 ? in[0] : 0, b1 = ln.y > 0 ? in[ln.x] : 0;
  cbase[g] = make_int2(b2, b1);
  unsigned short* out = col16 + cptr[g];
  for (int q = 0; q < ln.x + ln.y; ++q) {
    const int off = in[q] - (q < ln.x ? b2 : b1);
    if (off < 0 || off > 65535) *bad = 1;
    out[q] = (unsigned short)off;
  }
}

// fp32 copy of an operator's values (grid-stride)
__global__ void k_round_f32(const double* __restrict__ a, float* __restrict__ o, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    o[i] = (float)a[i];
}

// per step: the values of the item's row(s), in CSR order, into the node-blocked array (one warp per item,
// coalesced copies)
template <int D>
__global__ void k_nb_pack(const SysDesc* __restrict__ sys, const long long* __restrict__ item_off,
                          const long long* __restrict__ rowptr, const double* __restrict__ aout,
                          const long long* __restrict__ vptr, double* __restrict__ nbval,
                          float* __restrict__ nbval32) {
  const SysDesc S = sys[blockIdx.y];
  const int k = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (k >= S.n2 + S.n1) return;
  const long long g = item_off[blockIdx.y] + k;
  double* out = nbval + vptr[g];
  float* out32 = nbval32 ? nbval32 + vptr[g] : nullptr;
  auto put = [&](long long rb, long long re) {
    for (long long q = rb + lane; q < re; q += 32) {
      const double a = aout[q];
      out[q - rb] = a;
      if (out32) out32[q - rb] = (float)a;
    }
  };
  if (k < S.n2) {
    for (int a = 0; a < D; ++a) {
      const long long rb = rowptr[S.row_off + a * S.n2 + k], re = rowptr[S.row_off + a * S.n2 + k + 1];
      put(rb, re);
      out += re - rb;
      if (out32) out32 += re - rb;
    }
  } else {
    const long long row = S.row_off + D * S.n2 + (k - S.n2);
    put(rowptr[row], rowptr[row + 1]);
  }
}

// write-back of the conduit solution: u = z + s y (velocity), p = z + s y (pressure) on owned nodes.
template <int D>
__global__ void k_conduit_writeback(const SysDesc* __restrict__ sys, Level L, const double* __restrict__ z,
                                    const double* __restrict__ y, const double* __restrict__ s,
                                    const double* __restrict__ base, double* __restrict__ ecorr,
                                    double* __restrict__ out_u, double* __restrict__ out_p, int np0, int np1,
                                    int np2, long long n2_glob) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.n2 + S.n1) return;
  const long long o = S.row_off;
  const int npg[3] = {np0, np1, np2};
  int l[3] = {0, 0, 0}, g[3] = {0, 0, 0};
  if (r < S.n2) {
    unlex<D>(r, S.np, l);
    for (int a = 0; a < D; ++a) g[a] = 2 * S.c0[a] + l[a];
    const bool own = owns<D>(L, S, g);
    const long long gi = lex<D>(g, npg);
    for (int a = 0; a < D; ++a) {
      const long long k = o + a * S.n2 + r;
      const double full = z[k] + s[k] * y[k];
      if (own) out_u[a * n2_glob + gi] = full;
      if (ecorr) ecorr[k] = full - base[k];
    }
  } else {
    const int k1 = r - S.n2;
    const int shp1[3] = {S.nc[0] + 1, S.nc[1] + 1, S.nc[2] + 1};
    unlex<D>(k1, shp1, l);
    for (int a = 0; a < D; ++a) g[a] = 2 * (S.c0[a] + l[a]);
    if (!owns<D>(L, S, g)) return;
    int v[3];
    for (int a = 0; a < D; ++a) v[a] = g[a] / 2;
    const int shpg1[3] = {(npg[0] + 1) / 2, (npg[1] + 1) / 2, (npg[2] + 1) / 2};
    const long long k = o + D * S.n2 + k1;
    out_p[lex<D>(v, shpg1)] = z[k] + s[k] * y[k];
  }
}

}  // namespace lp
