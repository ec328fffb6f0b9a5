/*
 * lpfem.h -- C-ABI of the B200 local-parallel two-grid FEM hot path.
 *
 * Method: Algorithm 3 of arXiv 2311.05170 ("Local
 * parallel finite element algorithm"): per backward-Euler step
 *   Step 1  coarse decoupled marching on T_H          (eqs. pFFully..pcFully)
 *   Step 3  fine residual corrections on every
 *           overlapping subdomain Omega_j              (eqs. pFlocalFully,
 *                                                       pflocalFully, pmlocalFully, uclocalFully)
 *   Step 4  write-back of the core values D_j
 * for the transient triple-porosity / Navier-Stokes model with
 * Taylor-Hood P2-P1 in the conduit and P2 for the three porous pressures
 * (the paper's r = 1 case).  Readings of the paper where it is
 * silent are numbered C1..C25 in DESIGN.md; the ones that change an interface
 * are cited below.
 *
 * Conventions (all entry points):
 *  - Every pointer argument is borrowed for the duration of the call; inputs are
 *    deep-copied (including lpfem_coeffs.k_mult).  Output buffers are caller-owned.
 *  - Errors are returned as lpfem_status; no C++ exception crosses the ABI.
 *    lpfem_last_error() returns a ctx-owned message valid until the next call.
 *  - One host thread per ctx.  Work is enqueued on lpfem_dist.cuda_stream (NULL =
 *    the legacy default stream).  lpfem_create/step/get_fields/destroy are
 *    collective over lpfem_dist.world ranks (one process per GPU with the NCCL
 *    transport; with LPFEM_TRANSPORT_LOCAL all ranks live in one process and
 *    are stepped by lpfem_step_group).
 *  - Field layout: global lexicographic order, x fastest.  P2 fields live on the
 *    (2N_0+1)x(2N_1+1)[x(2N_2+1)] half-grid of their region (porous or conduit),
 *    P1 (conduit pressure) on the (N_0+1)x... vertices; the velocity is d
 *    consecutive component arrays (SoA).  Coordinates of half-grid point g are
 *    lo + g * ((hi - lo) / (2 N)) per axis (C21).
 *  - Arithmetic: fp64 throughout.
 */
#ifndef LPFEM_H
#define LPFEM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lpfem_ctx lpfem_ctx; /* opaque; owns all device memory */

typedef enum {
  LPFEM_OK = 0,
  LPFEM_EINVAL = 1,     /* bad pointer, size or parameter                                  */
  LPFEM_ENOTDIV = 2,    /* 1/h, 1/H or H/h not integral (relative tolerance 1e-12)            */
  LPFEM_EMISALIGN = 3,  /* subdomain grid does not divide the fine mesh / overlap not on h   */
  LPFEM_ENOCONV = 4,    /* Krylov or coarse Picard did not converge; the step is not committed */
  LPFEM_ECUDA = 5,      /* CUDA runtime error (message in lpfem_last_error)                */
  LPFEM_ENCCL = 6,      /* NCCL error (multi-GPU only)                                       */
  LPFEM_ENOMEM = 7,     /* device allocation failed                                          */
  LPFEM_ESTATE = 8      /* call out of order                                                 */
} lpfem_status;

enum { LPFEM_PROB_MMS = 0,       /* 2D: paper Ex1; 3D: Ex2 reflected z->1-z (C17) */
       LPFEM_PROB_INJECTION = 1, /* zero forcing, parabolic inflow on the conduit top face, no-slip sides (C16) */
       LPFEM_PROB_CONSTANT = 2,  /* p_i = c, u = 0, p = c/rho: an exact discrete steady state (invariant test)  */
       LPFEM_PROB_MMS_STEADY = 3 /* the MMS frozen at t = 0 (convergence tests)                                 */ };
enum { LPFEM_LAG_COMPOSITE = 0, /* e~^n from the written-back composite (mode B, default, C2) */
       LPFEM_LAG_SUBDOMAIN = 1  /* e~^n = the subdomain's own previous correction (mode A, C2) */ };

/* Geometry: two axis-aligned boxes sharing the full face Gamma normal to the last axis;
 * the conduit lies on the high side (BASELINE configs). */
typedef struct {
  int dim; /* 2 or 3 */
  double porous_lo[3], porous_hi[3], conduit_lo[3], conduit_hi[3];
} lpfem_geometry;

/* Coefficients.  Arrays are indexed 0 = matrix m, 1 = microfracture f, 2 = macrofracture F. */
typedef struct {
  double phi[3], C[3], k[3];
  double sigma, sigma_star, mu_tilde, nu, rho, alpha, eta;
  const double* k_mult; /* NULL, or one multiplier per porous COARSE cell (lexicographic, x fastest),
                           applied to k[0..2] and to k_F on Gamma (C15).  Deep-copied. */
} lpfem_coeffs;

typedef struct {
  int problem;        /* LPFEM_PROB_* */
  double inflow_peak; /* injection: peak inflow speed (1.0) */
  double const_value; /* constant problem: c */
} lpfem_data;

typedef struct {
  int lag_mode;         /* LPFEM_LAG_* */
  double krylov_rtol;   /* ||b - A x||_2 <= rtol ||b||_2 on every correction system (C19): 1e-12 */
  int max_iter;         /* per solve, counted in Krylov iterations: e.g. 20000 */
  int gmres_restart;    /* m of GMRES(m): 0 = the compiled length (45, measured best; LPFEM_GM at build
                           time); any other value than 0 or that length is LPFEM_EINVAL */
  double picard_rtol;   /* coarse NS: ||du||_2 <= rtol ||u||_2 (C11): 1e-13 */
  int picard_max;       /* 50 */
  int world_invariant;  /* 0 (default): Krylov launch geometry (thread-block cluster sizes, hence the order of
                           the dot-product reductions) chosen per rank for speed: fields agree across world
                           sizes to the solver tolerance (C19), not bitwise.  1: chosen from the GLOBAL system
                           counts, identical on every rank and for every world size, so the fields are bitwise
                           identical for any world (cost: at world N a rank's Krylov launches
                           use about 1/N of the SMs the per-rank choice would use) */
  int algorithm;        /* 3 (or 0, default): Algorithm 3, the local parallel method.
                           1: Algorithm 1, partitioned time stepping on the fine mesh T_h, the paper's
                           comparison scheme.  With H == h it runs on the dense coarse-step path (small meshes);
                           with H > h the subdomain grid must be 1 and the overlap 0: the whole regions are solved
                           by the fine stage's batched multilevel Krylov kernels (H sets the coarsest preconditioner
                           level), the Navier-Stokes step by Newton iterations to the C11 test */
} lpfem_opts;

enum { LPFEM_TRANSPORT_NCCL = 0,    /* one process per GPU; halo exchange by NCCL grouped send/recv (default) */
       LPFEM_TRANSPORT_LOCAL = 1    /* all ranks are contexts of ONE process (any devices, possibly the same one),
                                       stepped together by lpfem_step_group; the exchange copies each peer's
                                       packed send buffer (cudaMemcpyPeerAsync).  Same plan, pack/unpack and
                                       gather code as the NCCL transport; used to run the multi-rank path on
                                       a single GPU (tests) */ };

typedef struct {
  int rank, world, device;
  unsigned char nccl_id[128]; /* NCCL: from lpfem_nccl_unique_id on rank 0, broadcast by the caller.
                                 LOCAL: any 128 bytes identifying the group (equal on all its ranks) */
  void* cuda_stream;          /* cudaStream_t or NULL */
  int transport;              /* LPFEM_TRANSPORT_* */
} lpfem_dist;

typedef struct {
  long long steps;                 /* committed steps */
  long long fine_iters[2];         /* cumulative Krylov iterations: [porous PCG (sum over systems), conduit GMRES] */
  long long fine_max_iters[2];     /* max over systems in the last step */
  long long coarse_iters[2];       /* cumulative coarse iterations: [PCG, GMRES] */
  long long picard_iters;          /* cumulative coarse Picard iterations */
  double max_rel_residual[2];      /* last step, max over systems: [porous, conduit] */
  double t_coarse_ms, t_fine_ms;   /* cumulative device time of the coarse stage and of the fine stage */
  long long n_systems[2];          /* local systems on this rank: [porous (3 per subdomain), conduit] */
  long long n_rows[2], nnz[2];     /* local batched sizes: [porous family (per field), conduit family] */
  long long fine_dofs;             /* D of the metric: 3(2N+1)^d + d(2N+1)^d + (N+1)^d */
  long long kernel_launches;       /* cumulative launches of this library's kernels */
  double t_krylov_ms[2];           /* cumulative device time of the fine Krylov launches [PCG, GMRES] (CUDA events) */
  double bytes_krylov[2];          /* cumulative algorithmic bytes of those launches ("Roofline") */
  long long krylov_launches[2];    /* number of fine Krylov launches */
  long long coarse_factorizations; /* cumulative dense LU factorisations of the coarse Navier-Stokes Jacobian
                                      (chord iteration reuses the last one while it contracts) */
  double t_coarse_part_ms[3];      /* t_coarse_ms by part: [porous solves, Navier-Stokes chord/Picard iteration,
                                      coarse-box inverses of the multilevel preconditioner] (elapsed on the
                                      coarse stream; overlapped with the fine stage unless LPFEM_NO_OVERLAP) */
  long long h2d_bytes, d2h_bytes;  /* cumulative host->device / device->host bytes copied by this library
                                      (create: tables, patterns, k_mult; step: solver statistics, coarse
                                      Picard norms; get_fields: the fields when on_device = 0) */
} lpfem_stats;

/* NCCL unique id for a multi-GPU ctx (rank 0 only; world > 1). */
lpfem_status lpfem_nccl_unique_id(unsigned char out[128]);

/* Build meshes, subdomains (Algorithm 3 Step 2), patterns and the constant
 * operators; interpolate the initial state (C12).  H, h, overlap are lengths; 1/h, 1/H, H/h and
 * overlap/h must be integers and subdomain_grid[a] must divide the fine cells per axis of each
 * region (the grid applies per region, C8).  H == h selects Algorithm 1 on T_h: the coarse
 * step is then the fine step and every correction vanishes, so lpfem_step marches Algorithm 1 alone
 * (dense direct solves of the conduit system: meshes up to ~4e4 conduit DOFs).  Collective. */
lpfem_status lpfem_create(const lpfem_geometry* geom, const lpfem_coeffs* coeffs, const lpfem_data* data,
                          double H, double h, double overlap, const int subdomain_grid[3],
                          const lpfem_opts* opts, const lpfem_dist* dist, lpfem_ctx** out);

/* One step t_n -> t_{n+1} (C18: t_{n+1} = t_b + (n+1-n_b) dt, with (n_b, t_b) the step and time at which the
 * current dt took effect, i.e. (n+1) dt when dt never changes): coarse step, fine corrections on
 * every local subdomain, write-back and halo exchange.  A change
 * of dt re-assembles the dt-dependent operators.  Collective (world > 1: the convergence verdict is reduced
 * over the ranks, so all ranks commit or none does).
 * Commit semantics: the write-back goes to shadow composite arrays (and, in mode A, shadow corrections) that
 * replace the state only when every Krylov solve of every rank met C19 and the coarse step converged (C11).
 * On LPFEM_ENOCONV nothing is committed: lpfem_get_fields still returns t_n, lpfem_get_stats().steps is
 * unchanged, and the call may be repeated (e.g. with a smaller dt).  A non-converged coarse step that was
 * computed ahead on the side stream is reported by the step that consumes it.  Iteration and timing counters
 * in lpfem_stats are cumulative over all attempts.
 * The coarse step for t_{n+2} is computed on a side stream while this call's fine stage runs (it is
 * waited for at the next call); the fine Krylov solves start from the previous steps' corrections
 * (same stopping test, C19); the coarse Navier-Stokes solve is a chord iteration on the last factorised
 * Jacobian (same C11 test).  None of these changes the discrete solution beyond the stated tolerances. */
lpfem_status lpfem_step(lpfem_ctx* ctx, double dt);

/* lpfem_step for the ranks of one LPFEM_TRANSPORT_LOCAL group, stepped together from one host thread:
 * ctxs[0..n-1] are all `world` contexts of the group (any order).  Same semantics as lpfem_step on each
 * (the convergence verdict is the AND over the group).  LPFEM_EINVAL if the contexts do not form one complete
 * local group. */
lpfem_status lpfem_step_group(lpfem_ctx* const* ctxs, int n, double dt);

/* Fault injection (test hook, SURVEY 5 "failure detection"): cap the Krylov iterations of every later fine
 * solve of `family` (0 porous PCG, 1 conduit GMRES) at max_iter (> 0), so that the next steps fail with
 * LPFEM_ENOCONV; max_iter <= 0 removes the cap.  The coarse solves keep lpfem_opts.max_iter. */
lpfem_status lpfem_inject_fault(lpfem_ctx* ctx, int family, int max_iter);

/* Node counts of the global fine fields: [porous, conduit]. */
lpfem_status lpfem_get_sizes(const lpfem_ctx* ctx, long long n_nodes_p2[2], long long n_nodes_p1[2]);

/* Copy the composite fine fields at t_n: pF, pf, pm (n_p2[0] each), u (dim * n_p2[1], SoA), p (n_p1[1]).
 * on_device = 1: the pointers are device pointers on this ctx's GPU; 0: host pointers.  The
 * owned values of all ranks are gathered on `root` (other ranks may pass NULL).  Collective with the NCCL
 * transport; with LPFEM_TRANSPORT_LOCAL only the root's call is needed (it reads its peers' arrays). */
lpfem_status lpfem_get_fields(lpfem_ctx* ctx, double* pF, double* pf, double* pm, double* u, double* p,
                              int on_device, int root);

/* Copy the coarse state at t_n (same layout on the coarse mesh). */
lpfem_status lpfem_get_coarse_fields(lpfem_ctx* ctx, double* pF, double* pf, double* pm, double* u, double* p);

/* Mesh export for the bit-exact index check (C21, C22).  which = 2*level + region, level 0 coarse /
 * 1 fine, region 0 porous / 1 conduit.  coords: (n_p2, dim) half-grid node coordinates; cells:
 * (n_simplices, (dim+1)(dim+2)/2) P2 node indices per simplex (vertices in Kuhn order, then edge
 * midpoints); any pointer may be NULL.  n_out[0] = n_p2, n_out[1] = n_simplices. */
lpfem_status lpfem_get_mesh(const lpfem_ctx* ctx, int which, double* coords, int* cells, long long n_out[2]);

/* Subdomain layout of this rank: for each local system k (porous subdomains first, then conduit):
 * region, lexicographic position, core cells [c0, c1) and extended box cells [e0, e1) per axis.
 * Arrays hold n*3 ints each; n_out = number of local subdomains. */
lpfem_status lpfem_get_layout(const lpfem_ctx* ctx, int* region, int* pos, int* core0, int* core1, int* box0,
                              int* box1, int* n_out);

lpfem_status lpfem_get_stats(const lpfem_ctx* ctx, lpfem_stats* out);

/* Dump the last fine correction system of one local subdomain (debug / parity of a single solve):
 * family 0 porous (field 0 m, 1 f, 2 F), 1 conduit.  Writes nrows and nnz; if rowptr/col/val/rhs/x
 * are non-NULL they receive the CSR (rowptr nrows+1 int64, col nnz int32 local, val nnz), the RHS and
 * the solution.  Host pointers. */
lpfem_status lpfem_get_system(lpfem_ctx* ctx, int family, int local_index, int field, long long* nrows,
                              long long* nnz, long long* rowptr, int* col, double* val, double* rhs, double* x);

/* Measurement of the sparse matrix-vector product the Krylov kernels are built from (BASELINE metric
 * "SpMV % HBM peak"): y = A x over every fine system of one family (family 0 porous, the
 * three fields; 1 conduit, the current Oseen operators), with the same device routine (krylov.cuh
 * spmv_rows, same lanes per row) launched over all rows, `reps` times on the ctx stream; if flush != 0 a
 * 512 MiB buffer is written before every rep so each rep streams the matrix from HBM.  Returns the mean
 * device time per rep (CUDA events around the SpMV launch only) and the algorithmic bytes per rep:
 * 12 per nonzero (fp64 value + int32 column) + 8 per row pointer + 16 per row (x once, y).  Does not
 * change the solution state (reads the RHS vector, writes a Krylov work vector).  Host pointers. */
lpfem_status lpfem_bench_spmv(lpfem_ctx* ctx, int family, int reps, int flush, double* ms_per_rep,
                              double* bytes_per_rep);

/* Multi-GPU placement (host only, no device needed): rank_of_pos[s] for every subdomain position
 * s (lexicographic in the subdomain grid): LPT on the cell counts of the extended porous + conduit boxes
 * (csrc/halo.h).  n_cells_p / n_cells_c: fine cells per axis of the porous / conduit region. */
lpfem_status lpfem_placement(int dim, const int n_cells_p[3], const int n_cells_c[3], const int subdomain_grid[3],
                             int overlap_cells, int world, int* rank_of_pos);

/* Multi-GPU halo plan (host only): a fine node belongs to the rank of its owning subdomain (C3) under
 * lpfem_placement.  For region `region` (0 porous, 1 conduit), returns global node indices (P2 half-grid
 * lexicographic, or P1 vertex lexicographic if vertex_only): kind 0 = nodes owned by `peer` that `rank` reads
 * (its halo), 1 = nodes owned by `rank` that `peer` reads, 2 = all nodes owned by `peer`.  Sorted, unique.
 * out may be NULL to query the count. */
lpfem_status lpfem_halo_plan(int dim, const int n_cells_p[3], const int n_cells_c[3], const int subdomain_grid[3],
                             int overlap_cells, int region, int rank, int world, int vertex_only, int kind, int peer,
                             int* out, long long* n_out);

const char* lpfem_last_error(const lpfem_ctx* ctx);
const char* lpfem_status_string(lpfem_status s);
void lpfem_destroy(lpfem_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* LPFEM_H */
