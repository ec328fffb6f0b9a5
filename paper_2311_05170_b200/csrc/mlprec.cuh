// mlprec.cuh -- additive multilevel (BPX-type) preconditioner for the conduit saddle systems.
//
// For a fine conduit correction system on box Omega_j the right preconditioner is
//     M^-1 v = S_0 v + sum_{l=1}^{L-1} P_l S_l P_l^T v + P_L A_L^-1 P_L^T v
// where level l re-meshes the same box with the nested Kuhn mesh of size r_l h (r_l = 2, 4, ... dividing
// H/h), S_l is the block-diagonal scaling of that level's operator (velocity: 1/diag of the constant
// part; pressure: lumped-mass Schur approximation), and level L is the coarse mesh T_H restricted to the
// box with its full Newton-linearised operator inverted exactly (dense).  Because the meshes are nested and
// every form is integrated exactly, the re-discretised level operators equal the Galerkin products
// P_l^T A P_l (P:443-444 nesting).  P_l are the exact nodal prolongations (P2 velocity, P1 pressure)
// applied level by level; P_l^T is applied in two deterministic passes (per coarse cell, then per node).
// Fixed DOFs (dir / art velocity nodes, art pressure vertices; C4, C5) have zero scaling on every level.
#pragma once
#include "assembly.cuh"

namespace lp {

constexpr int NLMAX = 6;

struct MLArgs {
  int nl;                       // number of levels (intermediate + coarse); 0 = no multilevel part
  int q[NLMAX];                 // ratio of level l to level l-1 (level 0 = the fine system)
  const SysDesc* lsys[NLMAX];   // level boxes, one per system
  double* LR[NLMAX];            // restricted vectors (level row space)
  double* LZ[NLMAX];            // level corrections
  const double* LS[NLMAX];      // level scalings (0 on fixed rows)
  double* part;                 // restriction partials, per system at poff[sid]
  const long long* poff;
  const double* aci;            // dense inverses of the coarse-level systems (column-major), at aoff[sid]
  const long long* aoff;
  const SysDesc* fsys;          // fine boxes
  const double* s0;             // fine scaling (0 on fixed rows)
};

// P2 prolongation weights of a point g (box-local half-grid of the finer level) in the coarser level box
// (cells nc, ratio q): node codes within the coarse cell ({0,1,2}^D) and exact weights.
template <int D>
__device__ __forceinline__ void p2_weights(const int g[3], int q, const int nc[3], int cell[3], int code[n2_of(D)],
                                           double w[n2_of(D)]) {
  int num[3], ord[3] = {0, 1, 2};
  for (int a = 0; a < D; ++a) {
    cell[a] = min(g[a] / (2 * q), nc[a] - 1);
    num[a] = g[a] - 2 * q * cell[a];
  }
  for (int a = 1; a < D; ++a)
    for (int b = a; b > 0 && num[ord[b]] > num[ord[b - 1]]; --b) {
      int t = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = t;
    }
  long long lam[4];
  lam[0] = 2 * q - num[ord[0]];
  for (int k = 1; k < D; ++k) lam[k] = num[ord[k - 1]] - num[ord[k]];
  lam[D] = num[ord[D - 1]];
  int V[4][3];
  for (int a = 0; a < D; ++a) V[0][a] = 0;
  for (int k = 1; k <= D; ++k) {
    for (int a = 0; a < D; ++a) V[k][a] = V[k - 1][a];
    V[k][ord[k - 1]] += 2;
  }
  const double den = 2.0 * (double)q * (double)q;
  int n = 0;
  for (int k = 0; k <= D; ++k, ++n) {
    int c = 0, s = 1;
    for (int a = 0; a < D; ++a, s *= 3) c += V[k][a] * s;
    code[n] = c;
    w[n] = (double)(lam[k] * (lam[k] - q)) / den;
  }
  for (int a = 0; a <= D; ++a)
    for (int b = a + 1; b <= D; ++b, ++n) {
      int c = 0, s = 1;
      for (int e = 0; e < D; ++e, s *= 3) c += ((V[a][e] + V[b][e]) / 2) * s;
      code[n] = c;
      w[n] = (double)(2 * lam[a] * lam[b]) / den;
    }
}

template <int D>
__device__ __forceinline__ void p1_weights(const int g[3], int q, const int nc[3], int cell[3], int code[D + 1],
                                           double w[D + 1]) {
  int num[3], ord[3] = {0, 1, 2};
  for (int a = 0; a < D; ++a) {
    cell[a] = min(g[a] / (2 * q), nc[a] - 1);
    num[a] = g[a] - 2 * q * cell[a];
  }
  for (int a = 1; a < D; ++a)
    for (int b = a; b > 0 && num[ord[b]] > num[ord[b - 1]]; --b) {
      int t = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = t;
    }
  long long lam[4];
  lam[0] = 2 * q - num[ord[0]];
  for (int k = 1; k < D; ++k) lam[k] = num[ord[k - 1]] - num[ord[k]];
  lam[D] = num[ord[D - 1]];
  int V[3] = {0, 0, 0};
  for (int k = 0; k <= D; ++k) {
    if (k > 0) V[ord[k - 1]] += 2;
    int c = 0, s = 1;
    for (int a = 0; a < D; ++a, s *= 3) c += V[a] * s;
    code[k] = c;
    w[k] = (double)lam[k] / (2.0 * q);
  }
}

// coarse-level half-grid point of a cell-local code
template <int D>
__device__ __forceinline__ void code_point(int code, const int cell[3], int l[3]) {
  for (int a = 0; a < D; ++a) {
    l[a] = 2 * cell[a] + code % 3;
    code /= 3;
  }
}

// restriction pass 1: item = (coarse cell, component); partial sums of P^T src over the fine points the
// prolongation assigns to that cell.
template <int D>
__device__ void restrict_pass1(const SysDesc& SF, const SysDesc& SC, int q, const double* __restrict__ src,
                               double* __restrict__ part, int item) {
  constexpr int NCODE = p3_of(D);
  const int cidx = item / (D + 1), k = item % (D + 1);
  int c[3] = {0, 0, 0};
  unlex<D>(cidx, SC.nc, c);
  double acc[NCODE];
#pragma unroll
  for (int i = 0; i < NCODE; ++i) acc[i] = 0.0;
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  const int step = k < D ? 1 : 2;
  for (int a = 0; a < D; ++a) {
    lo[a] = 2 * q * c[a];
    hi[a] = 2 * q * c[a] + 2 * q - 1 + (c[a] == SC.nc[a] - 1 ? 1 : 0);
  }
  const int shp1[3] = {SF.nc[0] + 1, SF.nc[1] + 1, SF.nc[2] + 1};
  int g[3] = {0, 0, 0};
  for (g[2] = lo[2]; g[2] <= (D > 2 ? hi[2] : 0); g[2] += step)
    for (g[1] = lo[1]; g[1] <= hi[1]; g[1] += step)
      for (g[0] = lo[0]; g[0] <= hi[0]; g[0] += step) {
        int cell[3];
        if (k < D) {
          const double v = src[(long long)k * SF.n2 + lex<D>(g, SF.np)];
          if (v == 0.0) continue;
          int code[n2_of(D)];
          double w[n2_of(D)];
          p2_weights<D>(g, q, SC.nc, cell, code, w);
#pragma unroll
          for (int n = 0; n < n2_of(D); ++n) acc[code[n]] += w[n] * v;
        } else {
          int gv[3];
          for (int a = 0; a < D; ++a) gv[a] = g[a] >> 1;
          const double v = src[(long long)D * SF.n2 + lex<D>(gv, shp1)];
          if (v == 0.0) continue;
          int code[D + 1];
          double w[D + 1];
          p1_weights<D>(g, q, SC.nc, cell, code, w);
#pragma unroll
          for (int n = 0; n <= D; ++n) acc[code[n]] += w[n] * v;
        }
      }
  double* o = part + (long long)item * NCODE;
#pragma unroll
  for (int i = 0; i < NCODE; ++i) o[i] = acc[i];
}

// restriction pass 2: item = coarse row (velocity node x comp, then pressure vertex): sum the partials of
// the adjacent cells.
template <int D>
__device__ void restrict_pass2(const SysDesc& SC, const double* __restrict__ part, double* __restrict__ dst,
                               int row) {
  int l[3] = {0, 0, 0}, k;
  if (row < D * SC.n2) {
    k = row / SC.n2;
    unlex<D>(row % SC.n2, SC.np, l);
  } else {
    k = D;
    const int shp1[3] = {SC.nc[0] + 1, SC.nc[1] + 1, SC.nc[2] + 1};
    unlex<D>(row - D * SC.n2, shp1, l);
    for (int a = 0; a < D; ++a) l[a] *= 2;
  }
  int cand[3][2], ncand[3] = {1, 1, 1};
  for (int a = 0; a < D; ++a) {
    if (l[a] & 1) {
      cand[a][0] = (l[a] - 1) >> 1;
    } else {
      int n = 0;
      if ((l[a] >> 1) - 1 >= 0) cand[a][n++] = (l[a] >> 1) - 1;
      if ((l[a] >> 1) < SC.nc[a]) cand[a][n++] = l[a] >> 1;
      ncand[a] = n;
    }
  }
  double s = 0.0;
  for (int i2 = 0; i2 < (D > 2 ? ncand[2] : 1); ++i2)
    for (int i1 = 0; i1 < ncand[1]; ++i1)
      for (int i0 = 0; i0 < ncand[0]; ++i0) {
        int c[3] = {cand[0][i0], cand[1][i1], D > 2 ? cand[2][i2] : 0};
        int code = 0, m = 1;
        for (int a = 0; a < D; ++a, m *= 3) code += (l[a] - 2 * c[a]) * m;
        const long long item = lex<D>(c, SC.nc) * (D + 1) + k;
        s += part[item * p3_of(D) + code];
      }
  dst[row] = s;
}

// prolongation of a coarser-level vector src (box SC) to row `row` of the finer level box SF (ratio q)
template <int D>
__device__ __forceinline__ double prolong_row(const SysDesc& SF, const SysDesc& SC, int q,
                                              const double* __restrict__ src, int row) {
  int g[3] = {0, 0, 0}, cell[3];
  double s = 0.0;
  if (row < D * SF.n2) {
    const int k = row / SF.n2;
    unlex<D>(row % SF.n2, SF.np, g);
    int code[n2_of(D)];
    double w[n2_of(D)];
    p2_weights<D>(g, q, SC.nc, cell, code, w);
    const double* sk = src + (long long)k * SC.n2;
#pragma unroll
    for (int n = 0; n < n2_of(D); ++n) {
      if (w[n] == 0.0) continue;
      int l[3];
      code_point<D>(code[n], cell, l);
      s += w[n] * sk[lex<D>(l, SC.np)];
    }
  } else {
    const int shpf[3] = {SF.nc[0] + 1, SF.nc[1] + 1, SF.nc[2] + 1};
    unlex<D>(row - D * SF.n2, shpf, g);
    for (int a = 0; a < D; ++a) g[a] *= 2;
    int code[D + 1];
    double w[D + 1];
    p1_weights<D>(g, q, SC.nc, cell, code, w);
    const int shpc[3] = {SC.nc[0] + 1, SC.nc[1] + 1, SC.nc[2] + 1};
    const double* sp = src + (long long)D * SC.n2;
#pragma unroll
    for (int n = 0; n <= D; ++n) {
      if (w[n] == 0.0) continue;
      int l[3];
      code_point<D>(code[n], cell, l);
      for (int a = 0; a < D; ++a) l[a] >>= 1;
      s += w[n] * sp[lex<D>(l, shpc)];
    }
  }
  return s;
}

// ---------------------------------------------------------------------------------------------- host-side
// helpers (setup / per step)
__global__ void k_mask_from_scale(const double* __restrict__ s, double* __restrict__ m, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) m[i] = s[i] != 0.0 ? 1.0 : 0.0;
}

// dense column-major copies of the (masked, unscaled) coarse-level systems; fixed rows -> identity
__global__ void k_dense_batched(const SysDesc* __restrict__ sys, const long long* __restrict__ rowptr,
                                const int* __restrict__ col, const double* __restrict__ val,
                                const double* __restrict__ mask, const long long* __restrict__ aoff,
                                double* __restrict__ A) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  const int n = S.nrows;
  double* As = A + aoff[blockIdx.y];
  if (mask[S.row_off + r] == 0.0) {
    As[(long long)r * n + r] = 1.0;
    return;
  }
  for (long long q = rowptr[S.row_off + r]; q < rowptr[S.row_off + r + 1]; ++q)
    As[(long long)col[q] * n + r] = val[q];
}

// zero the rows and columns of fixed DOFs in the inverses (column-major)
__global__ void k_zero_fixed_inv(const SysDesc* __restrict__ sys, const double* __restrict__ mask,
                                 const long long* __restrict__ aoff, double* __restrict__ A) {
  const SysDesc S = sys[blockIdx.y];
  int j = blockIdx.x;  // column
  if (j >= S.nrows) return;
  const int n = S.nrows;
  double* As = A + aoff[blockIdx.y] + (long long)j * n;
  const bool fj = mask[S.row_off + j] == 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (fj || mask[S.row_off + i] == 0.0) As[i] = 0.0;
}

__global__ void k_set_identity(const SysDesc* __restrict__ sys, const long long* __restrict__ aoff,
                               double* __restrict__ B) {
  const SysDesc S = sys[blockIdx.y];
  int j = blockIdx.x;
  if (j >= S.nrows) return;
  const int n = S.nrows;
  double* Bs = B + aoff[blockIdx.y] + (long long)j * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) Bs[i] = i == j ? 1.0 : 0.0;
}

}  // namespace lp
