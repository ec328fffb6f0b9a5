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
// applied level by level; P_l^T is a stencil gather per coarse node (weights phi_I(x_g), Stencil).
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
  const double* aci;            // dense inverses of the coarse-level systems (row-major), at aoff[sid]
  const float* acif;            // same stored in fp32 (conduit): the preconditioner is then a different but
                                // fixed linear operator; right-preconditioned GMRES still meets C19 exactly
  const __nv_bfloat16* acib;    // experiment (LPFEM_ML_BF16): the same in bf16 (used instead of acif when set)
  const long long* aoff;
  const SysDesc* fsys;          // fine boxes
  const double* s0;             // fine scaling (0 on fixed rows)
  const struct Stencil* st[NLMAX];  // restriction stencils per level (ratio q[l]; direct mode: ratio r[l])
  int direct;                   // 1: every level restricts from / prolongs to the fine system directly;
                                // 2: level 0 from the fine system, levels 1.. directly from / to level 0
  const struct Stencil* st0[NLMAX];  // direct == 2: restriction stencils level 0 -> level l (ratio q0[l])
  int q0[NLMAX];                // direct == 2: ratio of level l to level 0
  int r[NLMAX];                 // ratio of level l to the fine mesh
  int nsub;                     // boxes per field: system sid = field * nsub + box
  long long lstride[NLMAX];     // field stride of the level vectors / scalings
  long long fstride;            // field stride of the fine scaling s0
  long long* phase;             // LPFEM_PHASE_TIMERS only: per-system sub-phase clocks (slots 8..15)
};

// Restriction P^T as a gather: the weight of coarse node I at fine point g is phi_I(x_g), so P^T v at a
// coarse node l is sum_delta phi(delta) v[q l + delta] over the fixed stencil of l's parity class, clipped at
// the box (points outside the box do not exist; the basis function values are cell-independent).
constexpr int STMAX = 24000;
struct Stencil {
  int q;
  int len[9];      // classes 0..2^D-1 (P2 nodes by half-grid parity), class 8 = P1 vertices
  int start[9];
  signed char off[STMAX][3];
  double w[STMAX];
};

// Barycentric coordinates of a point in its coarse cell: numerators num[a] (over 2q) sorted descending by a
// stable compare-exchange network (the Kuhn simplex containing the point, C22), with the axes they came from.
// Written without runtime-indexed arrays so that everything stays in registers (the previous insertion sort
// kept num/ord/V in local memory: ~600 local loads/stores in the 3D GMRES kernel).
template <int D>
__device__ __forceinline__ void kuhn_locate(const int g[3], int q, const int nc[3], int cell[3], long long lam[4],
                                            int vcode[4]) {
  int s0, s1 = 0, s2 = 0, o0 = 0, o1 = 1, o2 = 2;
  int num[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    cell[a] = min(g[a] / (2 * q), nc[a] - 1);
    num[a] = g[a] - 2 * q * cell[a];
  }
  s0 = num[0];
  s1 = num[1];
  s2 = num[2];
  auto cx = [](int& va, int& oa, int& vb, int& ob) {  // descending, stable (strict comparison)
    if (vb > va) {
      const int tv = va, to = oa;
      va = vb;
      oa = ob;
      vb = tv;
      ob = to;
    }
  };
  cx(s0, o0, s1, o1);
  if (D > 2) {
    cx(s1, o1, s2, o2);
    cx(s0, o0, s1, o1);
  }
  auto p3 = [](int o) { return o == 0 ? 1 : (o == 1 ? 3 : 9); };
  lam[0] = 2 * q - s0;
  if (D == 2) {
    lam[1] = s0 - s1;
    lam[2] = s1;
  } else {
    lam[1] = s0 - s1;
    lam[2] = s1 - s2;
    lam[3] = s2;
  }
  vcode[0] = 0;
  vcode[1] = 2 * p3(o0);
  vcode[2] = vcode[1] + 2 * p3(o1);
  if (D > 2) vcode[3] = vcode[2] + 2 * p3(o2);
}

// P2 prolongation weights of a point g (box-local half-grid of the finer level) in the coarser level box
// (cells nc, ratio q): node codes within the coarse cell ({0,1,2}^D) and exact weights.
template <int D>
__device__ __forceinline__ void p2_weights(const int g[3], int q, const int nc[3], int cell[3], int code[n2_of(D)],
                                           double w[n2_of(D)]) {
  long long lam[4];
  int vc[4];
  kuhn_locate<D>(g, q, nc, cell, lam, vc);
  const double inv = 1.0 / (2.0 * (double)q * (double)q);
  int n = 0;
#pragma unroll
  for (int k = 0; k <= D; ++k, ++n) {
    code[n] = vc[k];
    w[n] = (double)(lam[k] * (lam[k] - q)) * inv;
  }
#pragma unroll
  for (int a = 0; a <= D; ++a)
#pragma unroll
    for (int b = a + 1; b <= D; ++b, ++n) {
      code[n] = (vc[a] + vc[b]) / 2;  // midpoint of vertices a, b (digits 0/2 -> 0/1/2)
      w[n] = (double)(2 * lam[a] * lam[b]) * inv;
    }
}

template <int D>
__device__ __forceinline__ void p1_weights(const int g[3], int q, const int nc[3], int cell[3], int code[D + 1],
                                           double w[D + 1]) {
  long long lam[4];
  int vc[4];
  kuhn_locate<D>(g, q, nc, cell, lam, vc);
  const double inv = 1.0 / (2.0 * q);
#pragma unroll
  for (int k = 0; k <= D; ++k) {
    code[k] = vc[k];
    w[k] = (double)lam[k] * inv;
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

// 1/diag on free rows, 0 on fixed rows (level scalings and the fine Jacobi part of the porous preconditioner)
template <int D>
__global__ void k_porous_invdiag(const SysDesc* __restrict__ sys, Level L, const double* __restrict__ diag,
                                 double* __restrict__ dinv, double* __restrict__ mask, long long rows_total) {
  const SysDesc S = sys[blockIdx.y];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  int l[3] = {0, 0, 0};
  unlex<D>(r, S.np, l);
  const bool fixed = node_class<D>(L.G, S, l) >= CL_ART;
  for (int f = 0; f < 3; ++f) {
    const long long k = f * rows_total + S.row_off + r;
    dinv[k] = fixed ? 0.0 : 1.0 / diag[k];
    if (mask) mask[k] = fixed ? 0.0 : 1.0;
  }
}

// dense copies of the porous coarse-box systems, one per (field, box): system sid = field * nsub + box
__global__ void k_dense_porous(const SysDesc* __restrict__ sys, int nsub, const long long* __restrict__ rowptr,
                               const int* __restrict__ col, const double* __restrict__ val, long long nnz_total,
                               const double* __restrict__ mask, long long rows_total,
                               const long long* __restrict__ aoff, double* __restrict__ A) {
  const int sid = blockIdx.y, f = sid / nsub, b = sid % nsub;
  const SysDesc S = sys[b];
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= S.nrows) return;
  const int n = S.nrows;
  double* As = A + aoff[sid];
  if (mask[f * rows_total + S.row_off + r] == 0.0) {
    As[(long long)r * n + r] = 1.0;
    return;
  }
  for (long long q = rowptr[S.row_off + r]; q < rowptr[S.row_off + r + 1]; ++q)
    As[(long long)col[q] * n + r] = val[f * nnz_total + q];
}

__global__ void k_inv_rowmajor_porous(const SysDesc* __restrict__ sys, int nsub, const double* __restrict__ mask,
                                      long long rows_total, const long long* __restrict__ aoff,
                                      const double* __restrict__ Acm, double* __restrict__ Arm) {
  const int sid = blockIdx.y, f = sid / nsub, b = sid % nsub;
  const SysDesc S = sys[b];
  int i = blockIdx.x;
  if (i >= S.nrows) return;
  const int n = S.nrows;
  const double* m = mask + f * rows_total + S.row_off;
  const double* src = Acm + aoff[sid];
  double* dst = Arm + aoff[sid] + (long long)i * n;
  const bool fi = m[i] == 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) dst[j] = (fi || m[j] == 0.0) ? 0.0 : src[(long long)j * n + i];
}

__global__ void k_set_identity_n(const SysDesc* __restrict__ sys, int nsub, const long long* __restrict__ aoff,
                                 double* __restrict__ B) {
  const SysDesc S = sys[blockIdx.y % nsub];
  int j = blockIdx.x;
  if (j >= S.nrows) return;
  const int n = S.nrows;
  double* Bs = B + aoff[blockIdx.y] + (long long)j * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) Bs[i] = i == j ? 1.0 : 0.0;
}

// restriction by stencil gather.  Items are ordered class-major (component, parity class, node) so that
// neighbouring items walk the same stencil; each item's stencil is split over LN lanes (lane = 0..LN-1 of an
// aligned lane group) and reduced with shuffles, which cuts the dependent-load chain per row by LN.
template <int D, int NC, int LN, class ST>
__device__ __forceinline__ void restrict_item(const SysDesc& SF, const SysDesc& SC, const Stencil* __restrict__ T,
                                              const ST* __restrict__ src, double* __restrict__ dst, int item,
                                              int lane) {
  // every lane of the warp must reach the shuffles below: out-of-range items contribute nothing
  const bool valid = item < SC.nrows;
  if (!valid) item = 0;
  int l[3] = {0, 0, 0}, cls, row;
  const ST* sv;
  const int q = T->q;
  int shp[3];
  const int nvel = NC * SC.n2;
  if (item < nvel) {
    const int k = item / SC.n2;
    int rem = item - k * SC.n2;
    // parity classes in order 0..2^D-1; class kappa has prod_a (nc_a + 1 - kappa_a) nodes
    cls = 0;
    for (; cls < (1 << D); ++cls) {
      int cnt = 1;
      for (int a = 0; a < D; ++a) cnt *= SC.nc[a] + 1 - ((cls >> a) & 1);
      if (rem < cnt) break;
      rem -= cnt;
    }
    int ext[3] = {1, 1, 1};
    for (int a = 0; a < D; ++a) ext[a] = SC.nc[a] + 1 - ((cls >> a) & 1);
    int i3[3] = {0, 0, 0};
    unlex<D>(rem, ext, i3);
    for (int a = 0; a < D; ++a) l[a] = 2 * i3[a] + ((cls >> a) & 1);
    row = k * SC.n2 + (int)lex<D>(l, SC.np);
    sv = src + (long long)k * SF.n2;
    for (int a = 0; a < 3; ++a) shp[a] = SF.np[a];
  } else {
    const int shp1[3] = {SC.nc[0] + 1, SC.nc[1] + 1, SC.nc[2] + 1};
    unlex<D>(item - nvel, shp1, l);
    row = item;
    for (int a = 0; a < D; ++a) l[a] *= 2;
    cls = 8;
    sv = src + (long long)NC * SF.n2;
    for (int a = 0; a < 3; ++a) shp[a] = SF.nc[a] + 1;
  }
  const int b = T->start[cls], e = b + T->len[cls];
  const int sh = cls == 8 ? 1 : 0;
  int base[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) base[a] = q * l[a];
  double s0 = 0.0;
  // unconditional gathers: points outside the box are clamped onto it and weighted 0 (predicated loads were
  // chained one stencil entry at a time by the compiler)
#pragma unroll 4
  for (int i = b + lane; valid && i < e; i += LN) {
    int g0[3];
    bool ok0 = true;
    for (int a = 0; a < D; ++a) {
      g0[a] = base[a] + T->off[i][a];
      ok0 = ok0 && g0[a] >= 0 && g0[a] <= 2 * SF.nc[a];
      g0[a] = min(max(g0[a], 0), 2 * SF.nc[a]) >> sh;
    }
    const double v = (double)sv[lex<D>(g0, shp)];
    s0 += ok0 ? T->w[i] * v : 0.0;
  }
#pragma unroll
  for (int o = LN / 2; o > 0; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o, LN);
  if (valid && lane == 0) dst[row] = s0;
}

#ifndef LPFEM_RUNROLL
#define LPFEM_RUNROLL 2
#endif
constexpr int RUNROLL = LPFEM_RUNROLL;  // stencil entries per lane in flight in restrict_node

// restrict_item with the NC velocity components of a node in one item: items 0..SC.n2-1 are the coarse P2 nodes
// (class-major), items SC.n2.. the P1 vertices.  The stencil walk (class, offsets, clipping, index arithmetic) is
// shared by the components; every component's sum is the same ordered sum as restrict_item's (bitwise equal).
template <int D, int NC, int LN, class ST>
__device__ __forceinline__ void restrict_node(const SysDesc& SF, const SysDesc& SC, const Stencil* __restrict__ T,
                                              const ST* __restrict__ src, double* __restrict__ dst, int item,
                                              int lane) {
  const int nitems = SC.nrows - (NC - 1) * SC.n2;
  const bool valid = item < nitems;
  if (!valid) item = 0;
  int l[3] = {0, 0, 0}, cls, row;
  int shp[3];
  const int q = T->q;
  const bool vel = item < SC.n2;
  const ST* sv;
  if (vel) {
    int rem = item;
    cls = 0;
    for (; cls < (1 << D); ++cls) {
      int cnt = 1;
      for (int a = 0; a < D; ++a) cnt *= SC.nc[a] + 1 - ((cls >> a) & 1);
      if (rem < cnt) break;
      rem -= cnt;
    }
    int ext[3] = {1, 1, 1};
    for (int a = 0; a < D; ++a) ext[a] = SC.nc[a] + 1 - ((cls >> a) & 1);
    int i3[3] = {0, 0, 0};
    unlex<D>(rem, ext, i3);
    for (int a = 0; a < D; ++a) l[a] = 2 * i3[a] + ((cls >> a) & 1);
    row = (int)lex<D>(l, SC.np);
    sv = src;
    for (int a = 0; a < 3; ++a) shp[a] = SF.np[a];
  } else {
    const int shp1[3] = {SC.nc[0] + 1, SC.nc[1] + 1, SC.nc[2] + 1};
    unlex<D>(item - SC.n2, shp1, l);
    row = NC * SC.n2 + item - SC.n2;
    for (int a = 0; a < D; ++a) l[a] *= 2;
    cls = 8;
    sv = src + (long long)NC * SF.n2;
    for (int a = 0; a < 3; ++a) shp[a] = SF.nc[a] + 1;
  }
  const long long cs = vel ? SF.n2 : 0;  // component stride (P1 items read their one component NC times)
  const int b = T->start[cls], e = b + T->len[cls];
  const int sh = cls == 8 ? 1 : 0;
  int base[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) base[a] = q * l[a];
  double s[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) s[k] = 0.0;
#pragma unroll RUNROLL
  for (int i = b + lane; valid && i < e; i += LN) {
    int g0[3];
    bool ok0 = true;
    for (int a = 0; a < D; ++a) {
      g0[a] = base[a] + T->off[i][a];
      ok0 = ok0 && g0[a] >= 0 && g0[a] <= 2 * SF.nc[a];
      g0[a] = min(max(g0[a], 0), 2 * SF.nc[a]) >> sh;
    }
    const long long id = lex<D>(g0, shp);
    const double w = T->w[i];
    double v[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) v[k] = (double)sv[k * cs + id];
#pragma unroll
    for (int k = 0; k < NC; ++k) s[k] += ok0 ? w * v[k] : 0.0;
  }
#pragma unroll
  for (int o = LN / 2; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < NC; ++k) s[k] += __shfl_xor_sync(0xffffffffu, s[k], o, LN);
  if (valid && lane == 0) {
    if (vel) {
#pragma unroll
      for (int k = 0; k < NC; ++k) dst[k * SC.n2 + row] = s[k];
    } else {
      dst[row] = s[0];
    }
  }
}

// prolong_row for the NC velocity components of fine node nd at once (one location and weight evaluation for all
// components; each component's sum in prolong_row's order, bitwise equal)
template <int D, int NC>
__device__ __forceinline__ void prolong_node(const SysDesc& SF, const SysDesc& SC, int q, const double* __restrict__ src,
                                             int nd, double out[NC]) {
  int g[3] = {0, 0, 0}, cell[3];
  unlex<D>(nd, SF.np, g);
  int code[n2_of(D)];
  double w[n2_of(D)];
  p2_weights<D>(g, q, SC.nc, cell, code, w);
  int id[n2_of(D)];
#pragma unroll
  for (int n = 0; n < n2_of(D); ++n) {
    int l[3];
    code_point<D>(code[n], cell, l);
    id[n] = (int)lex<D>(l, SC.np);
  }
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    double v[n2_of(D)];
#pragma unroll
    for (int n = 0; n < n2_of(D); ++n) v[n] = src[k * SC.n2 + id[n]];
    double s = 0.0;
#pragma unroll
    for (int n = 0; n < n2_of(D); ++n)
      if (w[n] != 0.0) s += w[n] * v[n];
    out[k] = s;
  }
}

// prolongation of a coarser-level vector src (box SC) to row `row` of the finer level box SF (ratio q)
template <int D, int NC>
__device__ __forceinline__ double prolong_row(const SysDesc& SF, const SysDesc& SC, int q,
                                              const double* __restrict__ src, int row,
                                              const double* __restrict__ scl = nullptr) {
  int g[3] = {0, 0, 0}, cell[3];
  double s = 0.0;
  if (row < NC * SF.n2) {
    const int k = row / SF.n2;
    unlex<D>(row % SF.n2, SF.np, g);
    int code[n2_of(D)];
    double w[n2_of(D)];
    p2_weights<D>(g, q, SC.nc, cell, code, w);
    // unconditional gathers (every code lies in the coarse cell); zero weights add nothing
    double v[n2_of(D)];
#pragma unroll
    for (int n = 0; n < n2_of(D); ++n) {
      int l[3];
      code_point<D>(code[n], cell, l);
      const long long id = (long long)k * SC.n2 + lex<D>(l, SC.np);
      v[n] = scl ? scl[id] * src[id] : src[id];
    }
#pragma unroll
    for (int n = 0; n < n2_of(D); ++n)
      if (w[n] != 0.0) s += w[n] * v[n];
  } else {
    const int shpf[3] = {SF.nc[0] + 1, SF.nc[1] + 1, SF.nc[2] + 1};
    unlex<D>(row - NC * SF.n2, shpf, g);
    for (int a = 0; a < D; ++a) g[a] *= 2;
    int code[D + 1];
    double w[D + 1];
    p1_weights<D>(g, q, SC.nc, cell, code, w);
    const int shpc[3] = {SC.nc[0] + 1, SC.nc[1] + 1, SC.nc[2] + 1};
    double v[D + 1];
#pragma unroll
    for (int n = 0; n <= D; ++n) {
      int l[3];
      code_point<D>(code[n], cell, l);
      for (int a = 0; a < D; ++a) l[a] >>= 1;
      const long long id = (long long)NC * SC.n2 + lex<D>(l, shpc);
      v[n] = scl ? scl[id] * src[id] : src[id];
    }
#pragma unroll
    for (int n = 0; n <= D; ++n)
      if (w[n] != 0.0) s += w[n] * v[n];
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

// Batched in-place Gauss-Jordan inversion with partial pivoting, one CTA per matrix (column-major, n from
// the system descriptor).  Per pivot step: argmax reduction over the pivot column, row interchange, then the
// rank-1 update of all entries from the pivot row/column staged in shared memory.  The row interchanges are
// undone as column interchanges at the end (classic in-place Gauss-Jordan).  Used for the coarse-box
// operators of the multilevel preconditioner (n ~ 10^2 - 10^3).
template <int NT>
__global__ void __launch_bounds__(NT) k_gj_inverse(const SysDesc* __restrict__ sys, const long long* __restrict__ aoff,
                                                   double* __restrict__ Aall, int* __restrict__ perm_all) {
  extern __shared__ double sm[];
  const SysDesc S = sys[blockIdx.x];
  const int n = S.nrows;
  double* A = Aall + aoff[blockIdx.x];
  int* perm = perm_all + (aoff[blockIdx.x] / 1);  // scratch of length n inside a per-matrix region
  double* rowk = sm;          // n
  double* colk = sm + n;      // n
  __shared__ double rv[NT / 32];
  __shared__ int ri[NT / 32];
  __shared__ int piv_s;
  const int tid = threadIdx.x;
  for (int k = 0; k < n; ++k) {
    // pivot search in column k, rows k..n-1
    double best = -1.0;
    int bi = k;
    for (int i = k + tid; i < n; i += NT) {
      const double a = fabs(A[(long long)k * n + i]);
      if (a > best) {
        best = a;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      rv[tid >> 5] = best;
      ri[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double b2 = -1.0;
      int i2 = k;
      for (int w = 0; w < NT / 32; ++w)
        if (rv[w] > b2 || (rv[w] == b2 && ri[w] < i2)) {
          b2 = rv[w];
          i2 = ri[w];
        }
      piv_s = i2;
      perm[k] = i2;
    }
    __syncthreads();
    const int p = piv_s;
    if (p != k)
      for (int j = tid; j < n; j += NT) {
        const double t = A[(long long)j * n + k];
        A[(long long)j * n + k] = A[(long long)j * n + p];
        A[(long long)j * n + p] = t;
      }
    __syncthreads();
    const double d = A[(long long)k * n + k];
    const double dinv = d != 0.0 ? 1.0 / d : 0.0;
    for (int j = tid; j < n; j += NT) {
      rowk[j] = A[(long long)j * n + k];
      colk[j] = A[(long long)k * n + j];
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (int j = warp; j < n; j += NT / 32) {
      double* Aj = A + (long long)j * n;
      const double rj = rowk[j] * dinv;
      for (int i = lane; i < n; i += 32) {
        double v;
        if (i == k) v = j == k ? dinv : rj;
        else if (j == k) v = -colk[i] * dinv;
        else v = Aj[i] - colk[i] * rj;
        Aj[i] = v;
      }
    }
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, in reverse order
  for (int k = n - 1; k >= 0; --k) {
    const int p = perm[k];
    if (p != k)
      for (int i = tid; i < n; i += NT) {
        const double t = A[(long long)k * n + i];
        A[(long long)k * n + i] = A[(long long)p * n + i];
        A[(long long)p * n + i] = t;
      }
    __syncthreads();
  }
}

// row-major copy of the column-major inverses with the rows and columns of fixed DOFs zeroed
template <class T>
__device__ __forceinline__ T inv_cvt(double v) { return (T)v; }
template <>
__device__ __forceinline__ __nv_bfloat16 inv_cvt<__nv_bfloat16>(double v) { return __double2bfloat16(v); }

template <class T>
__global__ void k_inv_rowmajor(const SysDesc* __restrict__ sys, const double* __restrict__ mask,
                               const long long* __restrict__ aoff, const double* __restrict__ Acm,
                               T* __restrict__ Arm) {
  const SysDesc S = sys[blockIdx.y];
  int i = blockIdx.x;  // row
  if (i >= S.nrows) return;
  const int n = S.nrows;
  const double* src = Acm + aoff[blockIdx.y];
  T* dst = Arm + aoff[blockIdx.y] + (long long)i * n;
  const bool fi = mask[S.row_off + i] == 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    dst[j] = inv_cvt<T>((fi || mask[S.row_off + j] == 0.0) ? 0.0 : src[(long long)j * n + i]);
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
