// krylov.cuh -- batched Krylov solvers for the local correction systems.
//
// Design (B200): one thread-block cluster owns one linear system for the whole solve.  Every
// iteration runs inside a single kernel launch: the SpMV, the vector updates and the dot products
// are passes over the cluster's rows, and each reduction is a fixed-order warp-shuffle / shared
// memory / DSMEM sum, so results are deterministic and there is no host round trip.  Systems are
// independent (every subdomain correction reads only coarse data and its own lagged
// state), so the grid is simply (systems x cluster size).
//
//  * k_cg     conjugate gradients on the symmetrically Jacobi-scaled SPD porous systems
//             A~ = D^-1/2 A D^-1/2 (fixed rows/columns zero).  The stopping test uses the
//             unscaled residual ||b - A x||_2 = ||D^1/2 r~||_2 <= rtol ||b||_2 (C19) via the weights
//             w = diag(A); converged solves are re-checked with the true residual.
//  * k_gmres  restarted GMRES(M) with classical Gram-Schmidt and one re-orthogonalisation (CGS2),
//             Givens rotations, on the right-scaled saddle systems A' = mask A diag(s) (block-diagonal
//             preconditioner: velocity Jacobi, pressure mass Schur approximation).  Right
//             preconditioning keeps the residual of the original system, so the test
//             ||b - A x||_2 <= rtol ||b||_2 (C19) is exact; every restart recomputes it.
#pragma once
#include <cooperative_groups.h>
#include <type_traits>

#include "common.cuh"
#include "mlprec.cuh"

namespace lp {
namespace cgx = cooperative_groups;

// Matrix stream loads (values, column indices).  LPFEM_STREAM_LOADS=1 (experiment) uses the streaming cache hint
// (ld.global.cs, evict-first) so that the matrix would not push the gathered vector x out of the L2 -- measured
// much worse: the lanes of a row read the same 32-byte sectors at different times and evict-first re-fetched them
// (cfg4 NB SpMV 13.5 -> 24.3 GB of DRAM traffic per product, GMRES 5.2 -> 8.9 TB per step)
#ifndef LPFEM_BASIS_F32
#define LPFEM_BASIS_F32 1
#endif
#ifndef LPFEM_ZW_F32
#define LPFEM_ZW_F32 0
#endif
#ifndef LPFEM_NB_PREFETCH
#define LPFEM_NB_PREFETCH 0  // experiment: node-blocked SpMV, L2 bulk prefetch this many rounds ahead
#endif
#ifndef LPFEM_DOT16
#define LPFEM_DOT16 0
#endif
#ifndef LPFEM_NB_COLFIRST
#define LPFEM_NB_COLFIRST 1
#endif
#ifndef LPFEM_STREAM_LOADS
#define LPFEM_STREAM_LOADS 0
#endif
template <class T>
__device__ __forceinline__ T ldm(const T* p) {
#if LPFEM_STREAM_LOADS
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}

struct KSys {
  long long row_off;   // vectors: first row of this system in the family's vector row space
  long long prow_off;  // pattern: first row of this system in rowptr
  long long val_off;   // values: offset added to rowptr positions
  int nrows;
  int pad;
  long long item_off;  // node-blocked conduit format: first item (velocity node / pressure vertex) of the system
  int n2, n1;          // P2 nodes and P1 vertices of the system (conduit)
};

// Node-blocked conduit operator (fine Taylor-Hood systems): the D velocity rows of a P2 node share one column
// list, so they are stored together.  Item k of a system is velocity node k (k < n2) or pressure vertex k - n2.
//   node:   cols [L P2 neighbours (local P2 index) | L1 P1 neighbours (local P1 index)]; values: the node's D rows
//           consecutively, row a = [b = 0 block (L) | ... | b = D-1 block (L) | P1 block (L1)]  (the CSR row a
//           of the node, unchanged)
//   vertex: cols [L P2 neighbours]; values: the continuity row [b = 0 block (L) | ... | b = D-1 block]
// Per nonzero 8 B of value and, per (node, neighbour) pair, 4 B of column shared by the D x D block (the CSR
// stores 4 B per nonzero): 12 -> ~8.5 B per nonzero in 3D.
struct NBMat {
  const double* val;
  const float* val32;     // NULL, or the same values rounded to fp32 (the Arnoldi products of the multilevel GMRES)
  const int* col;
  const long long* vptr;  // per item (family item space): first value
  const long long* cptr;  // per item: first column
  const int2* len;        // per item: (L, L1)
  const unsigned short* col16;  // NULL, or the columns as 16-bit offsets from the item's bases (same positions)
  const int2* cbase;            // per item: (first P2 column, first P1 column); column = base + offset
};

struct KStat {
  int iters;
  int converged;
  double relres;  // final ||b - A x|| / ||b|| (true residual)
  long long vsum; // GMRES: sum over iterations of (j + 1), the basis vectors read per Gram-Schmidt pass
  long long spmv; // SpMV passes (iterations + residual checks)
};

// Optional per-phase timing of the GMRES iterations (build with -DLPFEM_PHASE_TIMERS): cluster rank 0,
// thread 0 of every system accumulates clock64() deltas per phase into A.phase[sid * 16 + k].
#ifdef LPFEM_PHASE_TIMERS
#define PHASE(k)                                                        \
  do {                                                                  \
    if (threadIdx.x == 0 && crank == 0) {                               \
      long long t_ = clock64();                                         \
      A.phase[sid * 16 + (k)] += t_ - tph;                              \
      tph = t_;                                                         \
    }                                                                   \
  } while (0)
#else
#define PHASE(k) \
  do {           \
  } while (0)
#endif

#ifdef LPFEM_PHASE_TIMERS
#define SUBPHASE(k)                                                                 \
  do {                                                                              \
    if (threadIdx.x == 0 && cgx::this_cluster().block_rank() == 0 && P.phase) {     \
      long long t_ = clock64();                                                     \
      P.phase[sid * 16 + 8 + (k)] += t_ - tsub;                                     \
      tsub = t_;                                                                    \
    }                                                                               \
  } while (0)
#else
#define SUBPHASE(k) \
  do {              \
  } while (0)
#endif

struct KArgs {
  const KSys* sys;
  const long long* rowptr;
  const int* col;
  const double* val;
  const double* b;
  const double* w;   // CG: residual-norm weights (diag of the unscaled operator); unused by GMRES
  double* x;
  double* r;
  double* p;         // CG: search direction; GMRES: W work vector
  double* q;         // CG: A p
  double* V;         // GMRES basis, (M+1) x rows_total
  long long rows_total;
  double rtol;
  int maxit;
  KStat* stat;
  long long* phase;  // LPFEM_PHASE_TIMERS only
  double reorth2;    // GMRES: reorthogonalise when ||w'||^2 < reorth2 ||w||^2 (Kahan-Parlett: 0.5)
  int smem_cols;     // 1: every CTA stages its rows' pattern (row offsets + column indices) in shared memory
  int warm;          // 1: x holds the previous step's solution of the same system, used as the initial guess;
                     // 2: also xp holds the one before: initial guess 2 x - xp (linear extrapolation in time)
  double* xp;        // warm == 2: the solution two steps back (updated to the previous one)
  NBMat nb;          // GMRES: node-blocked operator (nb.val != NULL), else the CSR (rowptr, col, val)
  const float* val32;  // NULL, or the fp32 copy of val (same offsets) for the Arnoldi (GMRES) / p -> A p (PCG) products
  double rr_fac;       // PCG with val32: replace the recurrence residual by the true one (fp64) when its weighted
                       // norm^2 fell by this factor since the last replacement
  const int* order;  // NULL, or the system of each cluster in launch order (clusters are dispatched in index
                     // order: the systems expected to take longest start first, LPT; no effect on the numbers)
};

// Sparsity pattern of the CTA's rows [r0, r1): staged once per solve in dynamic shared memory when it fits (the
// pattern is fixed for the whole Krylov solve; the SpMV then issues the value load and the x gather together,
// one L2/HBM latency per batch instead of three dependent ones: rowptr -> col -> x).
struct CtaPattern {
  const long long* rp;  // global (system-offset rowptr), used when !sm
  const int* col;
  const double* val;
  const int* srp;       // shared: row offsets relative to q0, nr + 1 entries
  const int* scol;      // shared: column indices of the CTA's nonzeros
  const double* sval;   // val + q0
  bool sm;
  const float* val32;   // NULL, or the fp32 copy of val (the GMRES's Arnoldi products, 2D)
  const float* sval32;  // val32 + q0
};

// dyn_off: bytes of dynamic shared memory in front of the pattern (the GMRES Hessenberg matrix)
template <int NT>
__device__ __forceinline__ CtaPattern stage_pattern(const KArgs& A, const long long* rp, const double* val, int r0,
                                                    int r1, int dyn_off = 0, const float* val32 = nullptr) {
  extern __shared__ __align__(16) int lp_ksm[];
  CtaPattern P{rp, A.col, val, nullptr, nullptr, nullptr, A.smem_cols != 0, val32, nullptr};
  if (P.sm) {
    const long long q0 = rp[r0];
    const int nr = r1 - r0;
    int* srp = lp_ksm + dyn_off / 4;
    int* scol = srp + ((nr + 4) & ~3);
    for (int i = threadIdx.x; i <= nr; i += NT) srp[i] = (int)(rp[r0 + i] - q0);
    const long long nq = rp[r1] - q0;
    for (long long i = threadIdx.x; i < nq; i += NT) scol[i] = A.col[q0 + i];
    __syncthreads();
    P.srp = srp;
    P.scol = scol;
    P.sval = val + q0;
    P.sval32 = val32 ? val32 + q0 : nullptr;
  }
  return P;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT, int NV>
struct RedSmem {
  double red[NT / 32][NV];
  double cred[2][NV];
  double fin[NV];
};

// Sum over the cluster of per-warp partials already stored in S.red[warp][0..n); returns via S.fin.
// Stage 1: value k is reduced by warp k mod (NT/32) with a butterfly over the per-warp partials (lane w reads
// red[w][k]); stage 2: thread k < n reads the cluster's CTA sums through DSMEM, all loads issued before the
// fixed-order sum.  Deterministic (fixed order everywhere), two short latency chains instead of 32 + CL serial
// loads on one thread.
template <int NT, int NV>
__device__ __forceinline__ void cluster_sum(RedSmem<NT, NV>& S, int n, int& par) {
  static_assert(NT / 32 <= 32, "one lane per warp partial");
  cgx::cluster_group cl = cgx::this_cluster();
  __syncthreads();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int k = warp; k < n; k += NT / 32) {
    double v = lane < NT / 32 ? S.red[lane][k] : 0.0;
    v = warp_sum(v);
    if (lane == 0) S.cred[par][k] = v;
  }
  cl.sync();
  if (tid < n) {
    const int nb = (int)cl.num_blocks();
    double t[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) t[k] = k < nb ? cl.map_shared_rank(&S.cred[par][0], k)[tid] : 0.0;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += t[k];
    S.fin[tid] = s;
  }
  __syncthreads();
  par ^= 1;
}

template <int NT, int NV>
__device__ __forceinline__ void put_partial(RedSmem<NT, NV>& S, int k, double v) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5][k] = v;
}

// y[i] = sum_q val[q] x[col[q]] for rows [r0, r1), TPR lanes per row.  Each lane issues its (col, val) loads
// in batches of U independent loads before the dependent x gathers, so that enough bytes are in flight per SM
// to cover the HBM latency (Little's law: ~45 KB per SM at ~1 us).
template <int NT, int TPR, class MT = double>
__device__ __forceinline__ void spmv_rows(const long long* __restrict__ rp, const int* __restrict__ col,
                                          const MT* __restrict__ val, const double* __restrict__ x,
                                          double* __restrict__ y, int r0, int r1) {
  constexpr int U = 8;
  const int lane = threadIdx.x % TPR;
  const int grp = threadIdx.x / TPR;
  constexpr int NG = NT / TPR;
  for (int base = r0; base < r1; base += NG) {
    const int r = base + grp;
    double s = 0.0;
    if (r < r1) {
      const long long qb = rp[r], qe = rp[r + 1];
      // Loads are unconditional, the index clamped to the row's last entry (an L1 hit) and its weight zeroed:
      // with predicated loads the compiler chained col -> x -> FMA one entry at a time (2-3 loads in flight per
      // thread, measured 3 TB/s on cfg4); unconditional loads let all 3U loads of a batch issue back to back.
      for (long long q0 = qb + lane; q0 < qe; q0 += (long long)TPR * U) {
        int cc[U];
        double vv[U], xx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const long long q = min(q0 + (long long)u * TPR, qe - 1);
          cc[u] = ldm(col + q);
          vv[u] = (double)ldm(val + q);
        }
        // a warp barrier between the (col, val) loads and the x gathers keeps the compiler from interleaving
        // them (it otherwise schedules for 32 registers and chains col -> x per entry)
        __syncwarp(__activemask());
#pragma unroll
        for (int u = 0; u < U; ++u) xx[u] = x[cc[u]];
        // zero the weights of clamped entries, then a pairwise tree (independent products, short chain)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (q0 + (long long)u * TPR >= qe) vv[u] = 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) vv[u] *= xx[u];
#pragma unroll
        for (int w = U / 2; w > 0; w >>= 1)
#pragma unroll
          for (int u = 0; u < w; ++u) vv[u] += vv[u + w];
        s += vv[0];
      }
    }
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, TPR);
    if (r < r1 && lane == 0) y[r] = s;
  }
}

// Software-pipelined variant: while the x gathers of row r are in flight, the (col, val) batch of row r + NG and
// the row pointers of row r + 2 NG are already loading (three stages), so the loads of a thread never wait on
// one another; rows longer than TPR * U finish their extra batches inline.  Same sums as spmv_rows per batch.
template <int NT, int TPR, int U, class MT = double>
__device__ __forceinline__ void spmv_rows_pipe(const long long* __restrict__ rp, const int* __restrict__ col,
                                               const MT* __restrict__ val, const double* __restrict__ x,
                                               double* __restrict__ y, int r0, int r1) {
  constexpr int NG = NT / TPR;
  const int lane = threadIdx.x % TPR;
  int r = r0 + threadIdx.x / TPR;
  auto rowq = [&](int rr, long long& b, long long& e) {
    if (rr < r1) {
      b = rp[rr];
      e = rp[rr + 1];
    } else {
      b = 0;
      e = 0;
    }
  };
  auto load = [&](long long q0, long long e, int* cc, MT* vv) {
    if (q0 - lane < e) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long q = min(q0 + (long long)u * TPR, e - 1);
        cc[u] = ldm(col + q);
        vv[u] = ldm(val + q);
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        cc[u] = 0;
        vv[u] = (MT)0;
      }
    }
  };
  auto batch = [&](long long q0, long long e, const int* cc, const MT* vm) {
    double xx[U], vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xx[u] = x[cc[u]];
#pragma unroll
    for (int u = 0; u < U; ++u) vv[u] = q0 + (long long)u * TPR < e ? (double)vm[u] * xx[u] : 0.0;
#pragma unroll
    for (int w = U / 2; w > 0; w >>= 1)
#pragma unroll
      for (int u = 0; u < w; ++u) vv[u] += vv[u + w];
    return vv[0];
  };
  long long b0, e0, b1, e1;
  rowq(r, b0, e0);
  rowq(r + NG, b1, e1);
  int cc[U];
  MT vv[U];
  load(b0 + lane, e0, cc, vv);
  for (int base = r0; base < r1; base += NG) {
    long long b2, e2;
    rowq(r + 2 * NG, b2, e2);
    int cn[U];
    MT vn[U];
    load(b1 + lane, e1, cn, vn);
    double s = 0.0;
    if (b0 < e0) {
      s = batch(b0 + lane, e0, cc, vv);
      for (long long q0 = b0 + lane + (long long)TPR * U; q0 < e0; q0 += (long long)TPR * U) {
        int c2[U];
        MT v2[U];
        load(q0, e0, c2, v2);
        s += batch(q0, e0, c2, v2);
      }
    }
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, TPR);
    if (r < r1 && lane == 0) y[r] = s;
    r += NG;
    b0 = b1;
    e0 = e1;
    b1 = b2;
    e1 = e2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cc[u] = cn[u];
      vv[u] = vn[u];
    }
  }
}

// same with the pattern staged in shared memory (row r of the system is srp[r - r0] .. srp[r - r0 + 1])
template <int NT, int TPR, class MT = double>
__device__ __forceinline__ void spmv_rows_sm(const int* __restrict__ srp, const int* __restrict__ scol,
                                             const MT* __restrict__ sval, const double* __restrict__ x,
                                             double* __restrict__ y, int r0, int r1) {
  constexpr int U = 8;
  const int lane = threadIdx.x % TPR;
  const int grp = threadIdx.x / TPR;
  constexpr int NG = NT / TPR;
  for (int base = r0; base < r1; base += NG) {
    const int r = base + grp;
    double s = 0.0;
    if (r < r1) {
      const int qb = srp[r - r0], qe = srp[r - r0 + 1];
      for (int q0 = qb + lane; q0 < qe; q0 += TPR * U) {
        double vv[U], xx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = min(q0 + u * TPR, qe - 1);  // unconditional loads (see spmv_rows)
          vv[u] = (double)ldm(sval + q);
          xx[u] = x[scol[q]];
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (q0 + u * TPR < qe) s += vv[u] * xx[u];
      }
    }
#pragma unroll
    for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, TPR);
    if (r < r1 && lane == 0) y[r] = s;
  }
}

// PIPE: software-pipelined rows (measured better for the porous PCG and the 2D conduit GMRES: cfg4 PCG 321 -> 278
// ms, cfg2 GMRES 167 -> 164 ms; worse for the 3D conduit GMRES: cfg3 99 -> 107 ms)
// lowp: multiply with the fp32 copy of the values when the pattern carries one (the GMRES's Arnoldi products)
template <int NT, int TPR, bool PIPE = true>
__device__ __forceinline__ void spmv(const CtaPattern& P, const double* __restrict__ x, double* __restrict__ y, int r0,
                                     int r1, bool lowp = false) {
  if (lowp && P.val32) {
    if (P.sm)
      spmv_rows_sm<NT, TPR, float>(P.srp, P.scol, P.sval32, x, y, r0, r1);
    else if (PIPE)
      spmv_rows_pipe<NT, TPR, 4, float>(P.rp, P.col, P.val32, x, y, r0, r1);
    else
      spmv_rows<NT, TPR, float>(P.rp, P.col, P.val32, x, y, r0, r1);
    return;
  }
  if (P.sm)
    spmv_rows_sm<NT, TPR>(P.srp, P.scol, P.sval, x, y, r0, r1);
  else if (PIPE)
    spmv_rows_pipe<NT, TPR, 4>(P.rp, P.col, P.val, x, y, r0, r1);
  else
    spmv_rows<NT, TPR>(P.rp, P.col, P.val, x, y, r0, r1);
}

// y = A x over the items [i0, i1) of one system (node-blocked format), TPR lanes per item; y rows of node i are
// a n2 + i, of vertex k: D n2 + k.  The lanes of an item walk its neighbours; per neighbour one column load, D
// (node) x gathers and D^2 value loads, all independent.
template <int NT, int TPR, int D, class MT = double, bool C16 = false, class XT = double>
__device__ __forceinline__ void spmv_nb(const NBMat& B, const MT* __restrict__ vals, long long item_off, int n2,
                                        const XT* __restrict__ x, double* __restrict__ y, int i0, int i1) {
  constexpr int NG = NT / TPR;
  const int lane = threadIdx.x % TPR;
  for (int base = i0; base < i1; base += NG) {
    const int it = base + threadIdx.x / TPR;
#if LPFEM_NB_PREFETCH
    // experiment: lane 0 of an item's group asks the L2 for the values and columns of the item this group takes
    // LPFEM_NB_PREFETCH rounds ahead (bulk prefetch: no registers or shared memory held while in flight).  The
    // range is widened to 16-byte bounds; the last item of the CTA's range is skipped so that the widened end stays
    // inside the next item's data.
    if (!C16 && lane == 0) {
      const int itp = it + LPFEM_NB_PREFETCH * NG;
      if (itp + 1 < i1) {
        const long long gp = item_off + itp;
        const int2 lp = B.len[gp];
        const bool nd = itp < n2;
        const unsigned long long v0 = (unsigned long long)(vals + B.vptr[gp]);
        const unsigned long long v1 = v0 + sizeof(MT) * (size_t)(nd ? D * (D * lp.x + lp.y) : D * lp.x);
        const unsigned long long c0 = (unsigned long long)(B.col + B.cptr[gp]);
        const unsigned long long c1 = c0 + 4ull * (size_t)(nd ? lp.x + lp.y : lp.x);
        const unsigned long long va = v0 & ~15ull, ca = c0 & ~15ull;
        const unsigned vb = (unsigned)(((v1 + 15ull) & ~15ull) - va), cbb = (unsigned)(((c1 + 15ull) & ~15ull) - ca);
        if (vb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(va), "r"(vb) : "memory");
        if (cbb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ca), "r"(cbb) : "memory");
      }
    }
#endif
    double acc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = 0.0;
    const bool node = it < n2;
    if (it < i1) {
      const long long g = item_off + it;
      const int2 ln = B.len[g];
      const MT* v = vals + B.vptr[g];
      const int* cl = C16 ? nullptr : B.col + B.cptr[g];
      const unsigned short* c16 = C16 ? B.col16 + B.cptr[g] : nullptr;
      const int2 cb = C16 ? B.cbase[g] : make_int2(0, 0);
      // column k of the item (P2 block: base cb.x; P1 block, positions >= L: base cb.y)
      auto colp2 = [&](int k) { return C16 ? cb.x + (int)ldm(c16 + k) : ldm(cl + k); };
      auto colp1 = [&](int k) { return C16 ? cb.y + (int)ldm(c16 + k) : ldm(cl + k); };
      const int L = ln.x, L1 = ln.y;
      if (node) {
        const int rl = D * L + L1;  // row length
#if LPFEM_NB_COLFIRST
        // all of the lane's P2 columns first (one latency for the whole item instead of one per neighbour), then
        // the gathers and values per neighbour
        constexpr int KMAX = (72 + TPR - 1) / TPR;
        int cc[KMAX];
#pragma unroll
        for (int t = 0; t < KMAX; ++t) cc[t] = lane + t * TPR < L ? colp2(lane + t * TPR) : 0;
#pragma unroll
        for (int t = 0; t < KMAX; ++t) {
          const int k = lane + t * TPR;
          if (k < L) {
            const int c = cc[t];
            double xb[D], vv[D][D];
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
              for (int bb = 0; bb < D; ++bb) vv[a][bb] = (double)ldm(v + a * rl + bb * L + k);
#pragma unroll
            for (int bb = 0; bb < D; ++bb) xb[bb] = (double)x[bb * n2 + c];
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
              for (int bb = 0; bb < D; ++bb) acc[a] += vv[a][bb] * xb[bb];
          }
        }
#else
        for (int k = lane; k < L; k += TPR) {
          const int c = colp2(k);
          double xb[D], vv[D][D];
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int bb = 0; bb < D; ++bb) vv[a][bb] = (double)ldm(v + a * rl + bb * L + k);
#pragma unroll
          for (int bb = 0; bb < D; ++bb) xb[bb] = (double)x[bb * n2 + c];
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int bb = 0; bb < D; ++bb) acc[a] += vv[a][bb] * xb[bb];
        }
#endif
        for (int k = lane; k < L1; k += TPR) {
          const int c = colp1(L + k);
          double vv[D];
#pragma unroll
          for (int a = 0; a < D; ++a) vv[a] = (double)ldm(v + a * rl + D * L + k);
          const double xp = (double)x[D * n2 + c];
#pragma unroll
          for (int a = 0; a < D; ++a) acc[a] += vv[a] * xp;
        }
      } else {
        for (int k = lane; k < L; k += TPR) {
          const int c = colp2(k);
          double vv[D], xb[D];
#pragma unroll
          for (int bb = 0; bb < D; ++bb) vv[bb] = (double)ldm(v + bb * L + k);
#pragma unroll
          for (int bb = 0; bb < D; ++bb) xb[bb] = (double)x[bb * n2 + c];
#pragma unroll
          for (int bb = 0; bb < D; ++bb) acc[0] += vv[bb] * xb[bb];
        }
      }
    }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int o = TPR / 2; o > 0; o >>= 1) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], o, TPR);
    if (it < i1 && lane == 0) {
      if (node) {
#pragma unroll
        for (int a = 0; a < D; ++a) y[a * n2 + it] = acc[a];
      } else {
        y[D * n2 + (it - n2)] = acc[0];
      }
    }
  }
}

// Standalone batched node-blocked SpMV over every system of the conduit family (lpfem_bench_spmv), fp64 or fp32 values
template <int NT, int TPR, int D, class MT>
__global__ void __launch_bounds__(NT) k_spmv_nb_family(const KSys* __restrict__ sys, NBMat B, const MT* vals,
                                                       const double* __restrict__ x, double* __restrict__ y,
                                                       int items_per_cta) {
  const KSys K = sys[blockIdx.y];
  const int i0 = blockIdx.x * items_per_cta;
  if (i0 >= K.n2 + K.n1) return;
  const int i1 = min(K.n2 + K.n1, i0 + items_per_cta);
  if (B.col16)
    spmv_nb<NT, TPR, D, MT, true>(B, vals, K.item_off, K.n2, x + K.row_off, y + K.row_off, i0, i1);
  else
    spmv_nb<NT, TPR, D, MT, false>(B, vals, K.item_off, K.n2, x + K.row_off, y + K.row_off, i0, i1);
}

// bytes of the GMRES(M) Hessenberg matrix (M + 1) x M in dynamic shared memory, 16-byte aligned
__host__ __device__ constexpr int gmres_h_bytes(int M) { return (((M + 1) * M * 8) + 15) & ~15; }

// Standalone batched SpMV over every system of a family (lpfem_bench_spmv): the Krylov kernels' row routine,
// grid (row blocks, systems).
template <int NT, int TPR, int PIPE_U, class MT = double>
__global__ void __launch_bounds__(NT) k_spmv_family(const KSys* __restrict__ sys, const long long* __restrict__ rowptr,
                                                    const int* __restrict__ col, const MT* __restrict__ val,
                                                    const double* __restrict__ x, double* __restrict__ y,
                                                    int rows_per_cta) {
  const KSys K = sys[blockIdx.y];
  const int r0 = blockIdx.x * rows_per_cta;
  if (r0 >= K.nrows) return;
  const int r1 = min(K.nrows, r0 + rows_per_cta);
  if (PIPE_U > 0)
    spmv_rows_pipe<NT, TPR, (PIPE_U > 0 ? PIPE_U : 1), MT>(rowptr + K.prow_off, col, val + K.val_off, x + K.row_off,
                                                          y + K.row_off, r0, r1);
  else
    spmv_rows<NT, TPR, MT>(rowptr + K.prow_off, col, val + K.val_off, x + K.row_off, y + K.row_off, r0, r1);
}

// ---------------------------------------------------------------------------------------------
template <int NT, int TPR>
__global__ void __launch_bounds__(NT, 1) k_cg(KArgs A) {
  cgx::cluster_group cl = cgx::this_cluster();
  const int CL = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const int sid = A.order ? A.order[blockIdx.x / CL] : blockIdx.x / CL;  // launch order: most work first
  const KSys K = A.sys[sid];
  const int chunk = (K.nrows + CL - 1) / CL;
  const int r0 = min(K.nrows, crank * chunk), r1 = min(K.nrows, r0 + chunk);
  const long long* rp = A.rowptr + K.prow_off;
  const int* col = A.col;
  const double* val = A.val + K.val_off;
  const double* b = A.b + K.row_off;
  const double* w = A.w + K.row_off;
  double* x = A.x + K.row_off;
  double* r = A.r + K.row_off;
  double* p = A.p + K.row_off;
  double* q = A.q + K.row_off;
  const CtaPattern PT = stage_pattern<NT>(A, rp, val, r0, r1);
  __shared__ RedSmem<NT, 2> S;
  int par = 0;
  const int tid = threadIdx.x;

  double pw = 0.0, pz = 0.0;
  for (int i = r0 + tid; i < r1; i += NT) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    p[i] = bi;
    pw += w[i] * bi * bi;
    pz += bi * bi;
  }
  put_partial(S, 0, pw);
  put_partial(S, 1, pz);
  cluster_sum(S, 2, par);
  const double bnorm = sqrt(S.fin[0]);
  double rz = S.fin[1];
  int it = 0, conv = 0, nspmv = 0;
  double relres = 0.0;
  if (bnorm == 0.0) {
    conv = 1;
  } else {
    const double tol2 = A.rtol * A.rtol * S.fin[0];
    int checks = 0;
    while (true) {
      cl.sync();  // p complete across the cluster
      spmv<NT, TPR>(PT, p, q, r0, r1);
      __syncthreads();
      double ppq = 0.0;
      for (int i = r0 + tid; i < r1; i += NT) ppq += p[i] * q[i];
      put_partial(S, 0, ppq);
      cluster_sum(S, 1, par);
      const double pq = S.fin[0];
      const double alpha = pq != 0.0 ? rz / pq : 0.0;
      double prr = 0.0, prz = 0.0;
      for (int i = r0 + tid; i < r1; i += NT) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        prr += w[i] * ri * ri;
        prz += ri * ri;
      }
      put_partial(S, 0, prr);
      put_partial(S, 1, prz);
      cluster_sum(S, 2, par);
      ++it;
      const double rrw = S.fin[0], rzn = S.fin[1];
      if (rrw <= tol2 || it >= A.maxit || pq == 0.0) {
        // verify with the true residual r = b - A x
        ++nspmv;
        cl.sync();
        spmv<NT, TPR>(PT, x, q, r0, r1);
        __syncthreads();
        double pt = 0.0, pzz = 0.0;
        for (int i = r0 + tid; i < r1; i += NT) {
          const double ri = b[i] - q[i];
          r[i] = ri;
          p[i] = ri;
          pt += w[i] * ri * ri;
          pzz += ri * ri;
        }
        put_partial(S, 0, pt);
        put_partial(S, 1, pzz);
        cluster_sum(S, 2, par);
        relres = sqrt(S.fin[0]) / bnorm;
        if (S.fin[0] <= tol2) {
          conv = 1;
          break;
        }
        if (it >= A.maxit || ++checks > 20 || pq == 0.0) break;
        rz = S.fin[1];
        continue;  // restart from the true residual
      }
      const double beta = rzn / rz;
      rz = rzn;
      for (int i = r0 + tid; i < r1; i += NT) p[i] = r[i] + beta * p[i];
    }
  }
  if (crank == 0 && tid == 0) {
    A.stat[sid].iters = it;
    A.stat[sid].converged = conv;
    A.stat[sid].relres = relres;
    A.stat[sid].vsum = 0;
    A.stat[sid].spmv = it + nspmv;
  }
  cl.sync();  // no CTA may exit while a peer still reads its shared memory (DSMEM, cluster_sum)
}

// ---------------------------------------------------------------------------------------------
// M^-1 v for the conduit systems (mlprec.cuh): fine diagonal + nested levels + exact coarse-box solve.
// v and Z are system-local fine vectors; work is spread over the whole cluster (gt, gs).
#ifndef LPFEM_RLN
#define LPFEM_RLN 4
#endif
constexpr int RLN = LPFEM_RLN;  // lanes per restricted row (4 vs 8: cfg2 GMRES 160 -> 153 ms, cfg1/cfg3 equal)

// all items of one level restriction, LN lanes per item, over the cluster's threads (gt of gs)
template <int D, int NC, int LN, class ST>
__device__ __forceinline__ void restrict_level(const SysDesc& SF, const SysDesc& SC, const Stencil* __restrict__ T,
                                               const ST* __restrict__ src, double* __restrict__ dst, int nitems,
                                               int gt, int gs) {
  const int wfirst = (gt & ~31) / LN;  // warp-uniform trip count (shuffles inside)
  for (int it = gt / LN, w0 = wfirst; w0 < nitems; it += gs / LN, w0 += gs / LN)
    restrict_node<D, NC, LN>(SF, SC, T, src, dst, it, gt % LN);
}

template <int D, int NC, class VIN = double, class ZT = double>
__device__ void apply_prec(const MLArgs& P, int sid, const VIN* __restrict__ v, ZT* __restrict__ Z, int r0,
                           int r1, int nrows) {
#ifdef LPFEM_PHASE_TIMERS
  long long tsub = clock64();
#endif
  cgx::cluster_group cl = cgx::this_cluster();
  const int gt = (int)cl.block_rank() * blockDim.x + threadIdx.x;
  const int gs = (int)cl.num_blocks() * blockDim.x;
  const int f = sid / P.nsub, bx = sid % P.nsub;
  const SysDesc S0 = P.fsys[bx];
  auto LRp = [&](int l) { return P.LR[l] + f * P.lstride[l] + P.lsys[l][bx].row_off; };
  auto LZp = [&](int l) { return P.LZ[l] + f * P.lstride[l] + P.lsys[l][bx].row_off; };
  auto LSp = [&](int l) { return P.LS[l] + f * P.lstride[l] + P.lsys[l][bx].row_off; };
  if (P.direct == 2) {
    // level 0 from the fine vector, then every coarser level directly from level 0 in one phase; coarse solve;
    // z_0 = S_0 r_0 + sum_{0<l<L} P_{0<-l} S_l r_l + P_{0<-L} z_L in one phase; fine combine.  Four cluster
    // barriers per application for any number of levels (the sequential chain needs 2 L + 2).
    {
      const SysDesc SC = P.lsys[0][bx];
      double* dst = LRp(0);
      const int wfirst = (gt & ~31) / RLN;
      for (int it = gt / RLN, w0 = wfirst; w0 < SC.nrows; it += gs / RLN, w0 += gs / RLN)
        restrict_item<D, NC, RLN>(S0, SC, P.st[0], v, dst, it, gt % RLN);
    }
    cl.sync();
    if (P.nl > 1) {
      const SysDesc SL0 = P.lsys[0][bx];
      int tot = 0;
      for (int l = 1; l < P.nl; ++l) tot += P.lsys[l][bx].nrows;
      const int wfirst = (gt & ~31) / RLN;
      for (int it = gt / RLN, w0 = wfirst; w0 < tot; it += gs / RLN, w0 += gs / RLN) {
        int l = 1, rem = it < tot ? it : tot - 1;
        while (rem >= P.lsys[l][bx].nrows) rem -= P.lsys[l++][bx].nrows;
        const SysDesc SC = P.lsys[l][bx];
        restrict_item<D, NC, RLN>(SL0, SC, P.st0[l], LRp(0), LRp(l), it < tot ? rem : SC.nrows, gt % RLN);
      }
      cl.sync();
    }
  } else if (P.direct) {
    // every level restricts the fine vector directly (one phase), coarse solve, one fused fine gather
    int tot = 0;
    for (int l = 0; l < P.nl; ++l) tot += P.lsys[l][bx].nrows;
    const int wfirst = (gt & ~31) / RLN;  // warp-uniform trip count (the lane groups of a warp shuffle together)
    for (int it = gt / RLN, w0 = wfirst; w0 < tot; it += gs / RLN, w0 += gs / RLN) {
      int l = 0, rem = it < tot ? it : tot - 1;
      while (rem >= P.lsys[l][bx].nrows) rem -= P.lsys[l++][bx].nrows;
      const SysDesc SC = P.lsys[l][bx];
      restrict_item<D, NC, RLN>(S0, SC, P.st[l], v, LRp(l), it < tot ? rem : SC.nrows, gt % RLN);
    }
    cl.sync();
  } else {
    SysDesc SF = S0;
    const double* src = nullptr;  // the previous level (level 0 restricts the input v)
    for (int l = 0; l < P.nl; ++l) {
      const SysDesc SC = P.lsys[l][bx];
      double* dst = LRp(l);
      const int nitems = SC.nrows - (NC - 1) * SC.n2;  // a node's NC components in one item
      if (l == 0) {
        restrict_level<D, NC, RLN>(SF, SC, P.st[l], v, dst, nitems, gt, gs);
      } else if (nitems * RLN * 2 <= gs) {
        // few items with long stencils (the coarse box, ratio H / (2h)): a warp per item, so that every thread
        // of the cluster walks a part of a stencil (RLN lanes per item left most threads idle)
        restrict_level<D, NC, 32>(SF, SC, P.st[l], src, dst, nitems, gt, gs);
      } else {
        restrict_level<D, NC, RLN>(SF, SC, P.st[l], src, dst, nitems, gt, gs);
      }
      SUBPHASE(2 * l);
      cl.sync();
      SUBPHASE(2 * l + 1);
      src = dst;
      SF = SC;
    }
  }
  if (P.nl > 0) {
    // exact coarse-box solve: LZ_L = A_L^-1 LR_L (row-major inverse, warp per row)
    const SysDesc SC = P.lsys[P.nl - 1][bx];
    const int n = SC.nrows;
    const double* rc = LRp(P.nl - 1);
    double* zc = LZp(P.nl - 1);
    const int lane = threadIdx.x & 31;
    if (P.acib) {
      const __nv_bfloat16* Ai = P.acib + P.aoff[sid];
      for (int i = gt >> 5; i < n; i += gs >> 5) {
        double s = 0.0;
#pragma unroll 4
        for (int j = lane; j < n; j += 32) s += (double)__bfloat162float(Ai[(long long)i * n + j]) * rc[j];
        s = warp_sum(s);
        if (lane == 0) zc[i] = s;
      }
    } else if (P.acif) {
      // CR rows per warp at once (CR independent row streams in flight per lane; rc[j] loaded once for all of
      // them); each row's sum in the same order as one row per warp
      constexpr int CR = 4;
      const float* Ai = P.acif + P.aoff[sid];
      for (int i0 = (gt >> 5) * CR; i0 < n; i0 += (gs >> 5) * CR) {
        double s[CR];
        const float* Ar[CR];
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          s[c] = 0.0;
          Ar[c] = Ai + (long long)min(i0 + c, n - 1) * n;  // rows past n repeat the last row (not stored)
        }
#pragma unroll 2
        for (int j = lane; j < n; j += 32) {
          const double rj = rc[j];
          float a[CR];
#pragma unroll
          for (int c = 0; c < CR; ++c) a[c] = Ar[c][j];
#pragma unroll
          for (int c = 0; c < CR; ++c) s[c] += (double)a[c] * rj;
        }
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          const double t = warp_sum(s[c]);
          if (lane == 0 && i0 + c < n) zc[i0 + c] = t;
        }
      }
    } else {
      const double* Ai = P.aci + P.aoff[sid];
      for (int i = gt >> 5; i < n; i += gs >> 5) {
        double s = 0.0;
#pragma unroll 4
        for (int j = lane; j < n; j += 32) s += Ai[(long long)i * n + j] * rc[j];
        s = warp_sum(s);
        if (lane == 0) zc[i] = s;
      }
    }
    SUBPHASE(6);
    cl.sync();
    if (P.direct == 2 && P.nl > 1) {
      const SysDesc SL0 = P.lsys[0][bx];
      const double* r0v = LRp(0);
      const double* s0v = LSp(0);
      double* z0 = LZp(0);
      for (int i = gt; i < SL0.nrows; i += gs) {
        double zi = s0v[i] * r0v[i];
        for (int l = 1; l < P.nl - 1; ++l)
          zi += prolong_row<D, NC>(SL0, P.lsys[l][bx], P.q0[l], LRp(l), i, LSp(l));
        zi += prolong_row<D, NC>(SL0, P.lsys[P.nl - 1][bx], P.q0[P.nl - 1], LZp(P.nl - 1), i);
        z0[i] = zi;
      }
      cl.sync();
    } else if (!P.direct) {
      for (int l = P.nl - 2; l >= 0; --l) {
        const SysDesc SL = P.lsys[l][bx];
        const SysDesc SU = P.lsys[l + 1][bx];
        const double* rl = LRp(l);
        const double* sl = LSp(l);
        const double* zu = LZp(l + 1);
        double* zl = LZp(l);
        // velocity nodes (NC components per item), then the P1 rows
        const int nitems = SL.nrows - (NC - 1) * SL.n2;
        for (int it = gt; it < nitems; it += gs) {
          if (it < SL.n2) {
            double pz[NC];
            prolong_node<D, NC>(SL, SU, P.q[l + 1], zu, it, pz);
#pragma unroll
            for (int k = 0; k < NC; ++k) {
              const int i = k * SL.n2 + it;
              zl[i] = sl[i] * rl[i] + pz[k];
            }
          } else {
            const int i = it + (NC - 1) * SL.n2;
            zl[i] = sl[i] * rl[i] + prolong_row<D, NC>(SL, SU, P.q[l + 1], zu, i);
          }
        }
        cl.sync();
      }
    }
  }
  SUBPHASE(7);
  const double* s0 = P.s0 + f * P.fstride + S0.row_off;
  if (NC > 1 && P.direct == 0) {
    // fine combine over the whole cluster, a node's NC velocity components per item (one location / weight
    // evaluation for all of them), then the P1 rows; Z is complete after the caller's cluster barrier
    const int nitems = S0.nrows - (NC - 1) * S0.n2;
    for (int it = gt; it < nitems; it += gs) {
      if (it < S0.n2) {
        double si[NC], zi[NC];
        bool any = false;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          si[k] = s0[k * S0.n2 + it];
          zi[k] = si[k] != 0.0 ? si[k] * (double)v[k * S0.n2 + it] : 0.0;
          any = any || si[k] != 0.0;
        }
        if (P.nl > 0 && any) {
          double pz[NC];
          prolong_node<D, NC>(S0, P.lsys[0][bx], P.q[0], LZp(0), it, pz);
#pragma unroll
          for (int k = 0; k < NC; ++k)
            if (si[k] != 0.0) zi[k] += pz[k];
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) Z[k * S0.n2 + it] = (ZT)zi[k];
      } else {
        const int i = it + (NC - 1) * S0.n2;
        const double si = s0[i];
        double zi = 0.0;
        if (si != 0.0) {
          zi = si * (double)v[i];
          if (P.nl > 0) zi += prolong_row<D, NC>(S0, P.lsys[0][bx], P.q[0], LZp(0), i);
        }
        Z[i] = (ZT)zi;
      }
    }
    return;
  }
  for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const double si = s0[i];
    double zi = 0.0;
    if (si != 0.0) {
      zi = si * (double)v[i];
      if (P.nl > 0) {
        if (P.direct == 1) {
          for (int l = 0; l < P.nl - 1; ++l)
            zi += prolong_row<D, NC>(S0, P.lsys[l][bx], P.r[l], LRp(l), i, LSp(l));
          zi += prolong_row<D, NC>(S0, P.lsys[P.nl - 1][bx], P.r[P.nl - 1], LZp(P.nl - 1), i);
        } else {
          zi += prolong_row<D, NC>(S0, P.lsys[0][bx], P.q[0], LZp(0), i);
        }
      }
    }
    Z[i] = (ZT)zi;
  }
  (void)nrows;
}

// ---------------------------------------------------------------------------------------------
// Preconditioned CG with the multilevel preconditioner (porous systems, SPD): unscaled masked operator,
// z = M^-1 r (symmetric: restriction = transpose of the prolongation), stopping test on the unscaled residual
// (C19) with the mask as weights.  One cluster per system; x, r, p, q, z are system-local.
template <int NT, int TPR, int D>
__global__ void __launch_bounds__(NT, 1) k_pcg_ml(KArgs A, MLArgs P, double* __restrict__ zbuf) {
  cgx::cluster_group cl = cgx::this_cluster();
  const int CL = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const int sid = A.order ? A.order[blockIdx.x / CL] : blockIdx.x / CL;  // launch order: most work first
  const KSys K = A.sys[sid];
  const int chunk = (K.nrows + CL - 1) / CL;
  const int r0 = min(K.nrows, crank * chunk), r1 = min(K.nrows, r0 + chunk);
  const long long* rp = A.rowptr + K.prow_off;
  const int* col = A.col;
  const double* val = A.val + K.val_off;
  const double* b = A.b + K.row_off;
  const double* w = A.w + K.row_off;
  double* x = A.x + K.row_off;
  double* r = A.r + K.row_off;
  double* p = A.p + K.row_off;
  double* q = A.q + K.row_off;
  double* z = zbuf + K.row_off;
  const CtaPattern PT = stage_pattern<NT>(A, rp, val, r0, r1, 0, A.val32 ? A.val32 + K.val_off : nullptr);
  // mixed precision: with an fp32 copy of the operator the products p -> A p use it; the recurrence residual then
  // drifts from b - A x at the fp32 level, so it is replaced by the true fp64 residual (and CG restarted) whenever
  // it fell by rr_fac (norm^2) since the last replacement, and the C19 test is always made on the true residual
  __shared__ RedSmem<NT, 2> S;
  int par = 0;
  const int tid = threadIdx.x;
  double pw = 0.0;
  double* xp = A.xp ? A.xp + K.row_off : nullptr;
  for (int i = r0 + tid; i < r1; i += NT) {
    const double bi = b[i];
    if (!A.warm) {
      x[i] = 0.0;
    } else if (xp) {
      const double xn = x[i];
      if (A.warm == 2) x[i] = 2.0 * xn - xp[i];
      xp[i] = xn;
    }
    r[i] = bi;
    pw += w[i] * bi * bi;
  }
  put_partial(S, 0, pw);
  cluster_sum(S, 1, par);
  const double bnorm = sqrt(S.fin[0]);
  const double tol2 = A.rtol * A.rtol * S.fin[0];
  int it = 0, conv = 0, nspmv = 0, checks = 0;
  double relres = 0.0, rz = 0.0;
  bool fresh = true;  // p must be restarted from z
  if (bnorm == 0.0) {
    conv = 1;
    for (int i = r0 + tid; i < r1; i += NT) x[i] = 0.0;
  } else if (A.warm) {
    // initial guess: the previous step's correction (the stopping test stays ||b - A x|| <= rtol ||b||, C19)
    spmv<NT, TPR>(PT, x, q, r0, r1);
    __syncthreads();
    double pt = 0.0;
    for (int i = r0 + tid; i < r1; i += NT) {
      const double ri = b[i] - q[i];
      r[i] = ri;
      pt += w[i] * ri * ri;
    }
    put_partial(S, 0, pt);
    cluster_sum(S, 1, par);
    ++nspmv;
    relres = sqrt(S.fin[0]) / bnorm;
    if (S.fin[0] <= tol2) conv = 1;
  }
  const bool lowp = A.val32 != nullptr;
  double rr_ref = lowp ? (A.warm ? relres * relres * bnorm * bnorm : bnorm * bnorm) : 0.0;
  while (!conv) {
    // z = M^-1 r, rz = r . z
    cl.sync();
    apply_prec<D, 1>(P, sid, r, z, r0, r1, K.nrows);
    double prz = 0.0;
    // vector passes two rows per round (independent loads of both rows in flight; the passes are latency-bound)
    {
      int i = r0 + tid;
      for (; i + NT < r1; i += 2 * NT) prz += r[i] * z[i] + r[i + NT] * z[i + NT];
      if (i < r1) prz += r[i] * z[i];
    }
    put_partial(S, 0, prz);
    cluster_sum(S, 1, par);
    const double rzn = S.fin[0];
    const double beta = fresh ? 0.0 : rzn / rz;
    rz = rzn;
    fresh = false;
    {
      int i = r0 + tid;
      for (; i + NT < r1; i += 2 * NT) {
        const double za = z[i], zb = z[i + NT], pa = p[i], pb = p[i + NT];
        p[i] = za + beta * pa;
        p[i + NT] = zb + beta * pb;
      }
      if (i < r1) p[i] = z[i] + beta * p[i];
    }
    cl.sync();
    spmv<NT, TPR>(PT, p, q, r0, r1, lowp);
    __syncthreads();
    double ppq = 0.0;
    {
      int i = r0 + tid;
      for (; i + NT < r1; i += 2 * NT) ppq += p[i] * q[i] + p[i + NT] * q[i + NT];
      if (i < r1) ppq += p[i] * q[i];
    }
    put_partial(S, 0, ppq);
    cluster_sum(S, 1, par);
    const double pq = S.fin[0];
    const double alpha = pq != 0.0 ? rz / pq : 0.0;
    double prr = 0.0;
    {
      int i = r0 + tid;
      for (; i + NT < r1; i += 2 * NT) {
        const double xa = x[i], xb = x[i + NT], pa = p[i], pb = p[i + NT];
        const double ra0 = r[i], rb0 = r[i + NT], qa = q[i], qb = q[i + NT], wa = w[i], wb = w[i + NT];
        x[i] = xa + alpha * pa;
        x[i + NT] = xb + alpha * pb;
        const double ra = ra0 - alpha * qa, rb = rb0 - alpha * qb;
        r[i] = ra;
        r[i + NT] = rb;
        prr += wa * ra * ra + wb * rb * rb;
      }
      if (i < r1) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        prr += w[i] * ri * ri;
      }
    }
    put_partial(S, 0, prr);
    cluster_sum(S, 1, par);
    ++it;
    if (S.fin[0] <= tol2 || it >= A.maxit || pq == 0.0 || (lowp && S.fin[0] <= A.rr_fac * rr_ref)) {
      ++nspmv;
      cl.sync();
      spmv<NT, TPR>(PT, x, q, r0, r1);
      __syncthreads();
      double pt = 0.0;
      for (int i = r0 + tid; i < r1; i += NT) {
        const double ri = b[i] - q[i];
        r[i] = ri;
        pt += w[i] * ri * ri;
      }
      put_partial(S, 0, pt);
      cluster_sum(S, 1, par);
      relres = sqrt(S.fin[0]) / bnorm;
      rr_ref = S.fin[0];
      if (S.fin[0] <= tol2) conv = 1;
      else if (it >= A.maxit || ++checks > 40 || pq == 0.0) break;
      else fresh = true;
    }
  }
  if (crank == 0 && tid == 0) {
    A.stat[sid].iters = it;
    A.stat[sid].converged = conv;
    A.stat[sid].relres = relres;
    A.stat[sid].vsum = 0;
    A.stat[sid].spmv = it + nspmv;
  }
  cl.sync();  // no CTA may exit while a peer still reads its shared memory (DSMEM, cluster_sum)
}

// ---------------------------------------------------------------------------------------------
// Dot products h_k = sum_i Vt_k[i] w[i] (k < nk) of the rows [r0, r1) into the per-warp partials S.red[.][k0+k],
// in chunks of 8 basis vectors (8 accumulators in registers; w is re-read once per chunk).  The 8 warp sums of
// a chunk are formed by a reduce-scatter butterfly (xor 4, 2, 1: lane l keeps value l & 7) followed by two
// shuffles across the lane octets: 9 shuffles per chunk instead of 8 x 5.  Fixed order: deterministic.
// ws: w is read as ws * w[i]; if pww != NULL the thread's sum of (ws w_i)^2 is added to *pww (first chunk)
template <int NT, int NV, class VT, class WT>
__device__ __forceinline__ void dots_chunked(RedSmem<NT, NV>& S, const VT* __restrict__ Vt, long long ld,
                                             const WT* __restrict__ w, int nk, int k0, int r0, int r1,
                                             double ws = 1.0, double* pww = nullptr) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const bool up4 = lane & 4, up2 = lane & 2, up1 = lane & 1;
#if LPFEM_DOT16
  // experiment: 16 basis vectors per pass, one row per round (the same 16 loads in flight; w read half as often)
  const bool up8 = lane & 8;
  for (int c0 = 0; c0 < nk; c0 += 16) {
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] = 0.0;
    double ww = 0.0;
    for (int i = r0 + threadIdx.x; i < r1; i += NT) {
      const double wi = ws * (double)w[i];
      VT va[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) va[u] = Vt[min(c0 + u, nk - 1) * ld + i];
#pragma unroll
      for (int u = 0; u < 16; ++u) acc[u] += c0 + u < nk ? (double)va[u] * wi : 0.0;
      ww += wi * wi;
    }
    if (pww && c0 == 0) *pww += ww;
    double a8[8], a4[4], a2[2];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double send = up8 ? acc[u] : acc[u + 8];
      a8[u] = (up8 ? acc[u + 8] : acc[u]) + __shfl_xor_sync(FULL, send, 8);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double send = up4 ? a8[u] : a8[u + 4];
      a4[u] = (up4 ? a8[u + 4] : a8[u]) + __shfl_xor_sync(FULL, send, 4);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double send = up2 ? a4[u] : a4[u + 2];
      a2[u] = (up2 ? a4[u + 2] : a4[u]) + __shfl_xor_sync(FULL, send, 2);
    }
    double a1 = (up1 ? a2[1] : a2[0]) + __shfl_xor_sync(FULL, up1 ? a2[0] : a2[1], 1);
    a1 += __shfl_xor_sync(FULL, a1, 16);
    if (lane < 16 && c0 + lane < nk) S.red[threadIdx.x >> 5][k0 + c0 + lane] = a1;
  }
  return;
#endif
  for (int c0 = 0; c0 < nk; c0 += 8) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    // two rows per round: 2 x 9 independent loads in flight per thread (the pass is latency-bound at one
    // 1024-thread CTA per SM)
    double ww = 0.0;
    int i = r0 + threadIdx.x;
    for (; i + NT < r1; i += 2 * NT) {
      const double wa = ws * (double)w[i], wb = ws * (double)w[i + NT];
      double va[8], vb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        va[u] = c0 + u < nk ? (double)Vt[(c0 + u) * ld + i] : 0.0;
        vb[u] = c0 + u < nk ? (double)Vt[(c0 + u) * ld + i + NT] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += va[u] * wa + vb[u] * wb;
      ww += wa * wa + wb * wb;
    }
    if (i < r1) {
      const double wi = ws * (double)w[i];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + u < nk) acc[u] += (double)Vt[(c0 + u) * ld + i] * wi;
      ww += wi * wi;
    }
    if (pww && c0 == 0) *pww += ww;
    double a4[4], a2[2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double send = up4 ? acc[u] : acc[u + 4];
      a4[u] = (up4 ? acc[u + 4] : acc[u]) + __shfl_xor_sync(FULL, send, 4);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double send = up2 ? a4[u] : a4[u + 2];
      a2[u] = (up2 ? a4[u + 2] : a4[u]) + __shfl_xor_sync(FULL, send, 2);
    }
    double a1 = (up1 ? a2[1] : a2[0]) + __shfl_xor_sync(FULL, up1 ? a2[0] : a2[1], 1);
    a1 += __shfl_xor_sync(FULL, a1, 8);
    a1 += __shfl_xor_sync(FULL, a1, 16);
    if (lane < 8 && c0 + lane < nk) S.red[threadIdx.x >> 5][k0 + c0 + lane] = a1;
  }
}

// sum_{k<n} c[k] Vt_k[i], loads issued in batches of 8 independent basis reads (one L2/HBM latency per batch
// instead of one per basis vector)
template <class VT>
__device__ __forceinline__ double basis_comb(const VT* __restrict__ V, long long ld, const double* c, int n,
                                             long long i) {
  double s = 0.0;
  for (int k0 = 0; k0 < n; k0 += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = (k0 + u < n) ? (double)V[(k0 + u) * ld + i] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < n) s += c[k0 + u] * v[u];
  }
  return s;
}

// the same for rows i and i + NT at once (loads of both rows in flight together)
template <int NT, class VT>
__device__ __forceinline__ void basis_comb2(const VT* __restrict__ V, long long ld, const double* c, int n,
                                            long long i, double& sa, double& sb) {
  sa = 0.0;
  sb = 0.0;
  for (int k0 = 0; k0 < n; k0 += 8) {
    double va[8], vb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      va[u] = (k0 + u < n) ? (double)V[(k0 + u) * ld + i] : 0.0;
      vb[u] = (k0 + u < n) ? (double)V[(k0 + u) * ld + i + NT] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < n) {
        sa += c[k0 + u] * va[u];
        sb += c[k0 + u] * vb[u];
      }
  }
}

// PC = false: right preconditioning folded into the matrix (A' = mask A diag(s)); the solution is y with
//             x = s y (applied at write-back).
// PC = true:  A is the masked unscaled operator and M^-1 = apply_prec; the solution is x itself.
// Arnoldi: classical Gram-Schmidt with the Kahan-Parlett "twice is enough" test: one pass computes V^T w and
// ||w||^2; ||w'||^2 = ||w||^2 - ||h||^2 decides whether a second projection is needed (||w'|| < ||w||/sqrt 2).
// The basis is stored unnormalised (Vt_k) with scales sig_k (v_k = sig_k Vt_k), so normalisation costs no pass.
template <int NT, int TPR, int M, int D, bool PC>
__global__ void __launch_bounds__(NT, 1) k_gmres(KArgs A, MLArgs P) {
  cgx::cluster_group cl = cgx::this_cluster();
  const int CL = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const int sid = A.order ? A.order[blockIdx.x / CL] : blockIdx.x / CL;  // launch order: most work first
  const KSys K = A.sys[sid];
  const int chunk = (K.nrows + CL - 1) / CL;
  const int r0 = min(K.nrows, crank * chunk), r1 = min(K.nrows, r0 + chunk);
  const long long* rp = A.rowptr + K.prow_off;
  const int* col = A.col;
  const double* val = A.val + K.val_off;
  const double* b = A.b + K.row_off;
  double* x = A.x + K.row_off;
  double* r = A.r + K.row_off;
  double* W = A.p + K.row_off;
  double* Zw = PC ? A.q + K.row_off : nullptr;
  const long long ld = A.rows_total;
  // Krylov basis: fp32 in the multilevel-preconditioned solves (PC), fp64 otherwise.  The basis is only the search
  // space: the Arnoldi relation then holds to fp32 accuracy, which bounds the reduction a restart cycle can reach
  // (~1e-7, against the ~1e-2..1e-3 the cycles achieve), and every restart recomputes the true residual in fp64,
  // so the C19 test ||b - A x|| <= rtol ||b|| stays exact.  Halves the Gram-Schmidt traffic.
  using VT = typename std::conditional<PC && LPFEM_BASIS_F32, float, double>::type;
  VT* V = reinterpret_cast<VT*>(A.V) + K.row_off;
  // Hessenberg matrix in dynamic shared memory (static shared memory is capped at 48 KB), pattern after it
  extern __shared__ __align__(16) double lp_gdyn[];
  double(*H)[M] = reinterpret_cast<double(*)[M]>(lp_gdyn);
  const CtaPattern PT = stage_pattern<NT>(A, rp, val, r0, r1, gmres_h_bytes(M), A.val32 ? A.val32 + K.val_off : nullptr);
  // node-blocked operator: the CTA's items (velocity nodes, then pressure vertices) instead of its rows; the
  // product then spans other CTAs' rows, so it ends with a cluster barrier
  const bool nbk = A.nb.val != nullptr;
  const int nitems = K.n2 + K.n1, ichunk = (nitems + CL - 1) / CL;
  const int it0 = min(nitems, crank * ichunk), it1 = min(nitems, it0 + ichunk);
  // lowp: the Arnoldi product of the multilevel GMRES multiplies with the fp32 copy of the operator when there is
  // one (mixed-precision GMRES: the restart's true residual b - A x below is always the fp64 operator, so the
  // C19 test stays exact; the fp32 operator only perturbs the search space, like the fp32 basis)
  auto matvec = [&](const double* X, double* Y, bool lowp = false) {
    if (nbk) {
      // (the 16-bit column experiment, NBMat::col16, is measured by the standalone SpMV only: compiling both column
      // paths into this 64-register kernel cost +13% GMRES time through register allocation alone)
      if (lowp && A.nb.val32)
        spmv_nb<NT, TPR, D, float, false>(A.nb, A.nb.val32, K.item_off, K.n2, X, Y, it0, it1);
      else
        spmv_nb<NT, TPR, D, double, false>(A.nb, A.nb.val, K.item_off, K.n2, X, Y, it0, it1);
      cl.sync();
    } else {
      spmv<NT, TPR, D == 2>(PT, X, Y, r0, r1, lowp);
      __syncthreads();
    }
  };
  __shared__ RedSmem<NT, M + 2> S;
  __shared__ double cs[M], sn[M], gv[M + 1], yv[M], hc[M + 1], sig[M + 1], hs[M + 1];
  int par = 0;
  const int tid = threadIdx.x;
#ifdef LPFEM_PHASE_TIMERS
  long long tph = clock64();
#endif

  double pb = 0.0;
  double* xp = A.xp ? A.xp + K.row_off : nullptr;
  for (int i = r0 + tid; i < r1; i += NT) {
    const double bi = b[i];
    if (!A.warm) {
      x[i] = 0.0;
    } else if (xp) {
      const double xn = x[i];
      if (A.warm == 2) x[i] = 2.0 * xn - xp[i];
      xp[i] = xn;
    }
    r[i] = bi;
    pb += bi * bi;
  }
  put_partial(S, 0, pb);
  cluster_sum(S, 1, par);
  const double bnorm = sqrt(S.fin[0]);
  double beta = bnorm;
  const double tol = A.rtol * bnorm;
  int it = 0, conv = 0, nspmv = 0;
  long long vsum = 0;
  if (bnorm == 0.0) {
    conv = 1;
    for (int i = r0 + tid; i < r1; i += NT) x[i] = 0.0;
  } else if (A.warm) {
    // initial guess: the previous step's correction (the stopping test stays ||b - A x|| <= rtol ||b||, C19)
    matvec(x, W);
    double pr = 0.0;
    for (int i = r0 + tid; i < r1; i += NT) {
      const double ri = b[i] - W[i];
      r[i] = ri;
      pr += ri * ri;
    }
    put_partial(S, 0, pr);
    cluster_sum(S, 1, par);
    ++nspmv;
    beta = sqrt(S.fin[0]);
    if (beta <= tol) conv = 1;
  }
  while (!conv) {
    for (int i = r0 + tid; i < r1; i += NT) V[i] = (VT)r[i];
    if (tid == 0) {
      sig[0] = 1.0 / beta;
      gv[0] = beta;
      for (int k = 1; k <= M; ++k) gv[k] = 0.0;
    }
    int jend = 0;
    for (int j = 0; j < M; ++j) {
      // Vt_0 (and the restart's sig/gv) must be complete across the cluster; for j > 0 the norm reduction that
      // closed iteration j - 1 (a cluster barrier after Vt_j was written) already guarantees it
      if (j == 0) cl.sync();
      PHASE(0);
      const double sj = sig[j];
      if constexpr (PC && LPFEM_ZW_F32 && D == 3) {
        // experiment: the preconditioned vector of the Arnoldi product in fp32 (node-blocked 3D only)
        if (nbk && A.nb.val32) {
          float* Zw32 = reinterpret_cast<float*>(Zw);
          apply_prec<D, D, VT, float>(P, sid, V + j * ld, Zw32, r0, r1, K.nrows);
          cl.sync();
          PHASE(1);
          spmv_nb<NT, TPR, D, float, false, float>(A.nb, A.nb.val32, K.item_off, K.n2, Zw32, W, it0, it1);
          cl.sync();
        } else {
          apply_prec<D, D>(P, sid, V + j * ld, Zw, r0, r1, K.nrows);
          cl.sync();
          PHASE(1);
          matvec(Zw, W, true);
        }
      } else if constexpr (PC) {
        apply_prec<D, D>(P, sid, V + j * ld, Zw, r0, r1, K.nrows);
        cl.sync();
        PHASE(1);
        matvec(Zw, W, true);
      } else {
        matvec(V + j * ld, W);
      }
      PHASE(2);
      // w = sj * W (applied on read, W is not rewritten);  pass A: h_k = sig_k Vt_k^T w and ||w||^2
      double pw = 0.0;
      dots_chunked<NT, M + 2>(S, V, ld, W, j + 1, 0, r0, r1, sj, &pw);
      put_partial(S, j + 1, pw);
      cluster_sum(S, j + 2, par);
      if (tid <= j) hc[tid] = S.fin[tid] * sig[tid];
      const double ww = S.fin[j + 1];
      __syncthreads();
      PHASE(3);
      // pass B: w' = w - sum_k h_k v_k, written as Vt_{j+1}; ||w'||^2
      VT* Vn = V + (j + 1) * ld;
      double pn = 0.0;
      if (tid <= j) hs[tid] = hc[tid] * sig[tid];
      __syncthreads();
      {
        int i = r0 + tid;
        for (; i + NT < r1; i += 2 * NT) {  // two rows per round (loads in flight)
          double ca, cb;
          basis_comb2<NT>(V, ld, hs, j + 1, i, ca, cb);
          const VT wa = (VT)(sj * W[i] - ca), wb = (VT)(sj * W[i + NT] - cb);
          Vn[i] = wa;
          Vn[i + NT] = wb;
          pn += (double)wa * (double)wa + (double)wb * (double)wb;  // the norm of the stored vector
        }
        if (i < r1) {
          const VT wv = (VT)(sj * W[i] - basis_comb(V, ld, hs, j + 1, i));
          Vn[i] = wv;
          pn += (double)wv * (double)wv;
        }
      }
      put_partial(S, 0, pn);
      cluster_sum(S, 1, par);
      double hn2 = S.fin[0];
      PHASE(4);
      if (hn2 < A.reorth2 * ww) {
        // second projection (CGS2): h2 = V^T w', w'' = w' - V h2
        __syncthreads();
        dots_chunked<NT, M + 2>(S, V, ld, Vn, j + 1, 0, r0, r1);
        cluster_sum(S, j + 1, par);
        double pn2 = 0.0;
        if (tid <= j) hs[tid] = S.fin[tid] * sig[tid] * sig[tid];
        __syncthreads();
        for (int i = r0 + tid; i < r1; i += NT) {
          double wi = (double)Vn[i];
          wi -= basis_comb(V, ld, hs, j + 1, i);
          const VT wv = (VT)wi;
          Vn[i] = wv;
          wi = (double)wv;
          pn2 += wi * wi;
        }
        if (tid <= j) hc[tid] += S.fin[tid] * sig[tid];
        __syncthreads();
        put_partial(S, 0, pn2);
        cluster_sum(S, 1, par);
        hn2 = S.fin[0];
      }
      PHASE(5);
      const double hn = sqrt(hn2);
      if (tid == 0) {
        sig[j + 1] = hn > 0.0 ? 1.0 / hn : 0.0;
        // apply the previous rotations to column j; the running entry stays in a register (the serial chain is
        // one rotation per step; cs, sn, hc loads are independent of it)
        double a = hc[0];
        for (int k = 0; k < j; ++k) {
          const double c = hc[k + 1];
          H[k][j] = cs[k] * a + sn[k] * c;
          a = -sn[k] * a + cs[k] * c;
        }
        H[j][j] = a;
        H[j + 1][j] = hn;
        const double c = hn;
        const double den = hypot(a, c);
        cs[j] = den > 0.0 ? a / den : 1.0;
        sn[j] = den > 0.0 ? c / den : 0.0;
        H[j][j] = den;
        H[j + 1][j] = 0.0;
        gv[j + 1] = -sn[j] * gv[j];
        gv[j] = cs[j] * gv[j];
      }
      __syncthreads();
      PHASE(6);
      ++it;
      vsum += j + 1;
      jend = j + 1;
      if (fabs(gv[j + 1]) <= tol || it >= A.maxit || hn == 0.0) break;
    }
    // y = H^-1 g (upper triangular, jend x jend)
    if (tid == 0) {
      for (int k = jend - 1; k >= 0; --k) {
        double s = gv[k];
        for (int m = k + 1; m < jend; ++m) s -= H[k][m] * yv[m];
        yv[k] = H[k][k] != 0.0 ? s / H[k][k] : 0.0;
      }
      for (int k = 0; k < jend; ++k) yv[k] *= sig[k];
    }
    __syncthreads();
    if (PC) {
      for (int i = r0 + tid; i < r1; i += NT) r[i] = basis_comb(V, ld, yv, jend, i);
      cl.sync();
      apply_prec<D, D>(P, sid, r, Zw, r0, r1, K.nrows);
      cl.sync();  // the fine combine writes Z over the whole cluster
      for (int i = r0 + tid; i < r1; i += NT) x[i] += Zw[i];
    } else {
      for (int i = r0 + tid; i < r1; i += NT) x[i] += basis_comb(V, ld, yv, jend, i);
    }
    cl.sync();
    ++nspmv;
    matvec(x, W);
    double pr = 0.0;
    for (int i = r0 + tid; i < r1; i += NT) {
      const double ri = b[i] - W[i];
      r[i] = ri;
      pr += ri * ri;
    }
    put_partial(S, 0, pr);
    cluster_sum(S, 1, par);
    beta = sqrt(S.fin[0]);
    if (beta <= tol) conv = 1;
    if (it >= A.maxit || beta == 0.0) break;
  }
  if (crank == 0 && tid == 0) {
    A.stat[sid].iters = it;
    A.stat[sid].converged = conv;
    A.stat[sid].relres = bnorm > 0.0 ? beta / bnorm : 0.0;
    A.stat[sid].vsum = vsum;
    A.stat[sid].spmv = it + nspmv;
  }
  cl.sync();  // no CTA may exit while a peer still reads its shared memory (DSMEM, cluster_sum)
}

}  // namespace lp
