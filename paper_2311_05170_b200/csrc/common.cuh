// common.cuh -- shared device/host definitions of the B200 lpfem library.
//
// Structured nested Kuhn meshes (C22): a region meshed with n[a] cells per axis; every
// cell is split into D! simplices  {x in cell : xi_pi0 >= xi_pi1 (>= xi_pi2)}  for each axis
// permutation pi, vertices V_0 = 0, V_k = sum_{t<k} e_{pi_t}.  P2 nodes live on the half-grid
// (2n+1 points per axis), P1 vertices on the even half-grid points.  Local P2 node order inside
// a simplex: vertices 0..D, then edge midpoints (a,b), a<b, lexicographic (C23).
//
// Paper: T_H and T_h regular, nested, compatible on Gamma; spaces of degree
// r+1 / r, here r = 1: Taylor-Hood P2-P1 and P2 pressures (BASELINE configs).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cmath>

#define HD __host__ __device__ __forceinline__

namespace lp {

constexpr int n2_of(int D) { return (D + 1) * (D + 2) / 2; }   // P2 nodes per simplex
constexpr int nt_of(int D) { return D == 1 ? 1 : (D == 2 ? 2 : 6); }  // Kuhn simplices per cell
constexpr int p3_of(int D) { return D == 1 ? 3 : (D == 2 ? 9 : 27); } // offset codes {0,1,2}^D
constexpr int ne_of(int D) { return D * (D + 1) / 2; }          // edges per simplex

// Kuhn tables for dimension 1..3, built on the host (mesh.cpp-equivalent code in lpfem.cu) and
// copied to __constant__ memory.
struct KuhnTables {
  int perm[6][3];            // axis permutation of each simplex type
  int pos[6][3];             // pos[t][axis] = rank of axis in perm[t]
  signed char off[6][10][3]; // half-grid offset (0,1,2) of local node i of type t
  signed char lookup[6][27]; // local node index of offset code o0 + 3 o1 + 9 o2, or -1
  int edge[6][2];            // edge k -> (a, b)
};

// Exact barycentric reference tensors (divided by |K|), built on the host by a Duffy-mapped
// Gauss-Legendre product rule that is exact for the degree-5 integrands ("Assembly").
template <int D>
struct RefT {
  static constexpr int N = n2_of(D), L = D + 1, NF = n2_of(D - 1), LF = D;
  double M22[N][N];            // int phi_i phi_j
  double G22[N][L][N][L];      // int dphi_i/dlam_k dphi_j/dlam_l
  double D12[L][N][L];         // int psi_m dphi_j/dlam_l
  double C3[N][N][N][L];       // int phi_i phi_m dphi_j/dlam_l
  double MF[NF][NF];           // facet (D-1 simplex): int phi_i phi_j
  double TF[NF][NF][LF];       // facet: int phi_i dphi_j/dlam_l
};

// One region (porous or conduit) at one level (coarse T_H or fine T_h).
struct LevelGeom {
  int n[3];        // cells per axis
  double lo[3], hi[3];
  double hc[3];    // cell size per axis, (hi - lo) / n
  double hg[3];    // half-grid step, (hi - lo) / (2 n)   (C21 coordinate formula)
  int R;           // cells of this level per coarse cell (1 on the coarse level)
  int far_g;       // half-grid index (last axis) of the Dirichlet face opposite Gamma
  int gamma_g;     // half-grid index (last axis) of Gamma
  int region;      // 0 porous, 1 conduit
};

// One local linear system: a fine subdomain box Omega_j (Algorithm 3 Step 2) or a
// whole coarse region (Step 1).  Cell ranges are in the level's cell grid.
struct SysDesc {
  int c0[3], nc[3];          // extended box: first cell and cells per axis
  int np[3];                 // P2 nodes per axis (2 nc + 1)
  int art_lo[3], art_hi[3];  // box face is artificial (interior to the region, C4)
  int pos[3];                // subdomain position in the subdomain grid (owner id per axis, C3)
  int n2, n1;                // P2 nodes and P1 vertices of the box
  int nrows;                 // rows of the system (porous: n2; conduit: D n2 + n1)
  int has_gamma;             // box touches Gamma
  int level;                 // 0 coarse, 1 fine
  long long row_off;         // first row in the family's row space
};

// Node classes, precedence dir > art > gamma > int (C4, C5).
enum { CL_INT = 0, CL_GAMMA = 1, CL_ART = 2, CL_DIR = 3 };

template <int D>
HD int node_class(const LevelGeom& G, const SysDesc& S, const int l[3]) {
  int g[3];
  for (int a = 0; a < D; ++a) g[a] = 2 * S.c0[a] + l[a];
  bool dir = g[D - 1] == G.far_g;
  for (int a = 0; a < D - 1; ++a) dir = dir || g[a] == 0 || g[a] == 2 * G.n[a];
  if (dir) return CL_DIR;
  for (int a = 0; a < D; ++a) {
    if (S.art_lo[a] && l[a] == 0) return CL_ART;
    if (S.art_hi[a] && l[a] == 2 * S.nc[a]) return CL_ART;
  }
  if (g[D - 1] == G.gamma_g) return CL_GAMMA;
  return CL_INT;
}

// Pressure vertex fixed (delta = 0) on the closure of the artificial faces: Q_0^h(Omega_j) (C4).
template <int D>
HD bool vertex_on_art(const SysDesc& S, const int l[3]) {
  for (int a = 0; a < D; ++a) {
    if (S.art_lo[a] && l[a] == 0) return true;
    if (S.art_hi[a] && l[a] == 2 * S.nc[a]) return true;
  }
  return false;
}

template <int D>
HD void unlex(long long r, const int* shape, int l[3]) {
  for (int a = 0; a < D; ++a) {
    l[a] = (int)(r % shape[a]);
    r /= shape[a];
  }
}

// 32-bit overload: row and node indices inside one box fit an int, and a 64-bit division by a runtime divisor is a
// ~70-instruction subroutine (the preconditioner's transfers unlex every row of every Krylov iteration)
template <int D>
HD void unlex(int r, const int* shape, int l[3]) {
  for (int a = 0; a < D; ++a) {
    const int q = r / shape[a];
    l[a] = r - q * shape[a];
    r = q;
  }
}

template <int D>
HD long long lex(const int l[3], const int* shape) {
  long long r = 0, s = 1;
  for (int a = 0; a < D; ++a) {
    r += (long long)l[a] * s;
    s *= shape[a];
  }
  return r;
}

// Gradients of the barycentric coordinates of Kuhn simplex type t with cell sizes h:
// lam_0 = 1 - xi_{pi0}, lam_k = xi_{pi(k-1)} - xi_{pi k}, lam_D = xi_{pi(D-1)}, xi_a = (x_a - o_a)/h_a.
template <int D>
HD void kuhn_grad(const int* perm, const double* h, double G[D + 1][D]) {
  for (int k = 0; k <= D; ++k)
    for (int a = 0; a < D; ++a) G[k][a] = 0.0;
  G[0][perm[0]] = -1.0 / h[perm[0]];
  for (int k = 1; k < D; ++k) {
    G[k][perm[k - 1]] += 1.0 / h[perm[k - 1]];
    G[k][perm[k]] -= 1.0 / h[perm[k]];
  }
  G[D][perm[D - 1]] = 1.0 / h[perm[D - 1]];
}

template <int D>
HD double kuhn_volume(const double* h) {
  double v = 1.0;
  for (int a = 0; a < D; ++a) v *= h[a];
  return D == 1 ? v : (D == 2 ? v * 0.5 : v / 6.0);
}

// ---------------------------------------------------------------------------------------------
// Forward-mode second-order jets over (x, y, z, t): value, gradient, symmetric Hessian.  Used to
// evaluate the manufactured solutions and derive their forcing from the strong form
// without hand-differentiation.
struct Jet {
  double v, g[4], H[4][4];
};

HD Jet jconst(double c) {
  Jet r;
  r.v = c;
  for (int i = 0; i < 4; ++i) {
    r.g[i] = 0.0;
    for (int j = 0; j < 4; ++j) r.H[i][j] = 0.0;
  }
  return r;
}
HD Jet jvar(double c, int k) {
  Jet r = jconst(c);
  r.g[k] = 1.0;
  return r;
}
HD Jet operator+(const Jet& a, const Jet& b) {
  Jet r;
  r.v = a.v + b.v;
  for (int i = 0; i < 4; ++i) {
    r.g[i] = a.g[i] + b.g[i];
    for (int j = 0; j < 4; ++j) r.H[i][j] = a.H[i][j] + b.H[i][j];
  }
  return r;
}
HD Jet operator-(const Jet& a, const Jet& b) {
  Jet r;
  r.v = a.v - b.v;
  for (int i = 0; i < 4; ++i) {
    r.g[i] = a.g[i] - b.g[i];
    for (int j = 0; j < 4; ++j) r.H[i][j] = a.H[i][j] - b.H[i][j];
  }
  return r;
}
HD Jet operator-(const Jet& a) { return jconst(0.0) - a; }
HD Jet operator*(const Jet& a, const Jet& b) {
  Jet r;
  r.v = a.v * b.v;
  for (int i = 0; i < 4; ++i) {
    r.g[i] = a.g[i] * b.v + a.v * b.g[i];
    for (int j = 0; j < 4; ++j)
      r.H[i][j] = a.H[i][j] * b.v + a.g[i] * b.g[j] + a.g[j] * b.g[i] + a.v * b.H[i][j];
  }
  return r;
}
HD Jet operator*(double c, const Jet& a) {
  Jet r;
  r.v = c * a.v;
  for (int i = 0; i < 4; ++i) {
    r.g[i] = c * a.g[i];
    for (int j = 0; j < 4; ++j) r.H[i][j] = c * a.H[i][j];
  }
  return r;
}
HD Jet operator+(double c, const Jet& a) {
  Jet r = a;
  r.v += c;
  return r;
}
HD Jet operator+(const Jet& a, double c) { return c + a; }
HD Jet operator-(double c, const Jet& a) { return c + (-a); }
HD Jet operator-(const Jet& a, double c) { return a + (-c); }
// f(a) with f, f', f'' at a.v
HD Jet jchain(const Jet& a, double f0, double f1, double f2) {
  Jet r;
  r.v = f0;
  for (int i = 0; i < 4; ++i) {
    r.g[i] = f1 * a.g[i];
    for (int j = 0; j < 4; ++j) r.H[i][j] = f1 * a.H[i][j] + f2 * a.g[i] * a.g[j];
  }
  return r;
}
HD Jet jsin(const Jet& a) { double s = sin(a.v), c = cos(a.v); return jchain(a, s, c, -s); }
HD Jet jcos(const Jet& a) { double s = sin(a.v), c = cos(a.v); return jchain(a, c, -s, -c); }
HD Jet jexp(const Jet& a) { double e = exp(a.v); return jchain(a, e, e, e); }

}  // namespace lp
