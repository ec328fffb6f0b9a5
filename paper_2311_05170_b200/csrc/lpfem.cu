// lpfem.cu -- context, setup (stage a0), the per-step driver of Algorithm 3 and the C-ABI.
//
// Paper: Algorithm 3.  Step 1 (coarse) runs redundantly on every GPU with
// the same kernels as the fine stage (one "system" per coarse region); Step 3 solves
// every local correction as a batch; Step 4 writes core values back.  See DESIGN.md.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <map>
#include <mutex>

#include <cub/device/device_scan.cuh>
#include <cusolverDn.h>
#include <nccl.h>

#include "../../include/lpfem.h"
#include "assembly.cuh"
#include "conduit.cuh"
#include "krylov.cuh"
#include "problem.cuh"
#include "tables.h"
#include "halo.h"

using namespace lp;

namespace {

struct Err : std::runtime_error {
  lpfem_status code;
  Err(lpfem_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      throw Err(LPFEM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +          \
                                 std::to_string(__LINE__));                                        \
  } while (0)

thread_local long long tl_launches = 0;  // kernel launches of this library (host thread of the ctx)
// host<->device bytes moved by this library (host thread of the ctx): lpfem_stats.h2d_bytes / d2h_bytes
thread_local long long tl_h2d = 0, tl_d2h = 0;
inline void count_copy(size_t n, cudaMemcpyKind k) {
  if (k == cudaMemcpyHostToDevice) tl_h2d += (long long)n;
  if (k == cudaMemcpyDeviceToHost) tl_d2h += (long long)n;
}
inline cudaError_t cpy(void* d, const void* s, size_t n, cudaMemcpyKind k) {
  count_copy(n, k);
  return cudaMemcpy(d, s, n, k);
}
inline cudaError_t cpya(void* d, const void* s, size_t n, cudaMemcpyKind k, cudaStream_t st) {
  count_copy(n, k);
  return cudaMemcpyAsync(d, s, n, k, st);
}
template <class T>
cudaError_t cpysym(const T& sym, const void* s, size_t n) {
  tl_h2d += (long long)n;
  return cudaMemcpyToSymbol(sym, s, n);
}
#define CKL()                      \
  do {                             \
    CK(cudaGetLastError());        \
    ++tl_launches;                 \
  } while (0)

template <class T>
T* dalloc(size_t n) {
  if (n == 0) n = 1;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) throw Err(LPFEM_ENOMEM, std::string("cudaMalloc ") + std::to_string(n * sizeof(T)) + " B: " + cudaGetErrorString(e));
  return (T*)p;
}

#ifndef LPFEM_GM
#define LPFEM_GM 45
#endif
#ifndef LPFEM_TPR2
#define LPFEM_TPR2 4
#endif
#ifndef LPFEM_TPR3
#define LPFEM_TPR3 8
#endif
// GMRES restart length (compile-time: shared-memory Hessenberg and reductions).  Measured (cfg1/2/3 max
// iterations 316/344/484 at 30 -> 246/313/399 at 45; GMRES time -1%/-10%/-14%)
constexpr int GM = LPFEM_GM;
#ifndef LPFEM_NTG
#define LPFEM_NTG 1024
#endif
constexpr int NTG = LPFEM_NTG;  // threads per CTA of the conduit GMRES
constexpr int TPR2 = LPFEM_TPR2, TPR3 = LPFEM_TPR3;  // conduit SpMV lanes per row (2D ~28 nnz/row, 3D ~93; 3D 8 vs 16:
                                                     // cfg4 GMRES 2169 -> 2145 ms)

// NCCL is loaded lazily (multi-GPU only) so that the library has no link-time NCCL dependency; in a torch
// process this resolves to the NCCL torch already loaded.
struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    send = (decltype(send))dlsym(h, "ncclSend");
    recv = (decltype(recv))dlsym(h, "ncclRecv");
    groupStart = (decltype(groupStart))dlsym(h, "ncclGroupStart");
    groupEnd = (decltype(groupEnd))dlsym(h, "ncclGroupEnd");
    errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    return getUniqueId && commInitRank && commDestroy && send && recv && groupStart && groupEnd && errStr && allReduce;
  }
};
NcclApi g_nccl;

#define CKN(call)                                                                                  \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) throw Err(LPFEM_ENCCL, std::string(#call) + ": " + g_nccl.errStr(r_));  \
  } while (0)

// device copy of one peer's index lists and exchange buffers
struct PeerX {
  int peer = -1;
  int np_give = 0, nc_give = 0, np_need = 0, nc_need = 0;
  int *give_p = nullptr, *give_c = nullptr, *need_p = nullptr, *need_c = nullptr;
  double *sbuf = nullptr, *rbuf = nullptr;
};

struct Family {
  int kind = 0;   // 0 porous (scalar P2, 3 fields), 1 conduit (Taylor-Hood saddle)
  int level = 1;  // 0 coarse, 1 fine
  std::vector<SysDesc> hs;
  SysDesc* ds = nullptr;
  long long rows = 0, nnz = 0;
  int maxrows = 0, maxitems = 0;
  long long* rowptr = nullptr;
  int* col = nullptr;
  // porous
  double *val = nullptr, *diag = nullptr, *isq = nullptr, *wn = nullptr, *dinv = nullptr, *zv = nullptr;
  // conduit
  double *aconst = nullptr, *aout = nullptr, *scale = nullptr, *mask = nullptr;
  // vectors
  double *base = nullptr, *z = nullptr, *lag = nullptr, *qf = nullptr, *aux = nullptr, *W = nullptr;
  double *rhs = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *V = nullptr, *ecorr = nullptr;
  double* ecorr2 = nullptr;  // mode A: corrections of the step being computed (committed by swapping with ecorr)
  std::vector<KSys> hk;
  KSys* dk = nullptr;
  KStat* dstat = nullptr;
  std::vector<KStat> hstat;
  // node-blocked copy of the fine conduit operator (krylov.cuh NBMat), used by the GMRES SpMV
  double* nbval = nullptr;
  float* nbval32 = nullptr;      // fp32 copy for the Arnoldi products (mixed-precision GMRES), NULL with LPFEM_NB_F64
  float* aout32 = nullptr;       // the same for the CSR operator of the fine conduit family without a node-blocked copy
  float* val32 = nullptr;        // fine porous family: fp32 copy of the 3 operators (mixed-precision PCG)
  int* ticket = nullptr;         // block counter of the persistent conduit assembly (k_conduit_step_w)
  int* nbcol = nullptr;
  unsigned short* nbcol16 = nullptr;  // 16-bit column offsets (experiment LPFEM_NB_COL16; NULL by default)
  int2* nbcbase = nullptr;
  long long *nbvptr = nullptr, *nbcptr = nullptr, *nbioff = nullptr;
  int2* nblen = nullptr;
  long long nb_items = 0, nb_ncols = 0;
  std::vector<long long> h_ioff;
  std::vector<int> order;        // fine Krylov launches: systems in decreasing expected work (rows x last iterations)
  int* dorder = nullptr;
  int cluster = 1;
  int nsys_rule = 1;             // system count the cluster rules use (local, or global with world_invariant)
  bool cluster_checked = false;  // cluster size reduced until all clusters are co-resident (resident_cluster)
  bool bandwidth_bound = false;  // large systems: keep the largest cluster even if the launch needs two waves
  int solved = 0;                // previous solutions held: x (>= 1), xp (>= 2) (Krylov warm start)
  double* xp = nullptr;          // the solution one step before x (extrapolated warm start)
  std::vector<long long> sys_nnz;        // nnz per Krylov system
  std::vector<long long> hrp;            // host copy of rowptr (CTA pattern sizes for the Krylov launches)
  std::vector<int> sub_region, sub_pos;  // per local subdomain (fine)
  std::vector<std::array<int, 3>> core0, core1;
  void free_all() {
    void* ptrs[] = {ds, rowptr, col, val, diag, isq, wn, dinv, zv, aconst, aout, scale, mask, base, z, lag, qf, aux, W,
                    rhs, x, r, p, q, V, ecorr, ecorr2, dk, dstat, xp, dorder, nbval, nbval32, aout32, val32, ticket, nbcol, nbcol16, nbcbase, nbvptr, nbcptr,
                    nbioff, nblen};
    for (void* ptr : ptrs)
      if (ptr) cudaFree(ptr);
  }
};

}  // namespace

struct lpfem_ctx {
  int D = 2;
  lpfem_geometry geom{};
  Coef co{};
  ProbData pd{};
  lpfem_opts opts{};
  lpfem_dist dist{};
  double H = 0, h = 0;
  int R = 1, ov = 0, m[3] = {1, 1, 1};
  int nf_p[3] = {1, 1, 1}, nf_c[3] = {1, 1, 1}, nc_p[3] = {1, 1, 1}, nc_c[3] = {1, 1, 1};
  Level Lp[2], Lc[2];  // [level] porous, conduit
  Family fam[2][2];    // [level][kind]
  // coarse state [old/new]
  // coarse state ring: slot n % 3 holds t_n (Step 1 runs one step ahead on the side stream st2)
  double* cst[3][3] = {};
  double* cu[3] = {};
  double* cp[3] = {};
  cudaStream_t st2 = nullptr;  // coarse marching stream (overlaps the fine stage), highest priority
  int prio_hi = 0;
  int nsm = 148;               // SMs of the device
  cudaStream_t st3 = nullptr;  // fine porous stage, concurrent with the fine conduit stage (independent)
  cudaEvent_t evp[3] = {};     // fork / join of st3; [2]: conduit GMRES about to launch (gates the porous PCG)
  cudaStream_t st4 = nullptr;  // split GMRES launch (experiment LPFEM_GM_SPLIT): the light systems' launch
  cudaEvent_t evs[2] = {};     // fork / join of st4
  int gm_split[3] = {0, 0, 0}; // LPFEM_GM_SPLIT=k:c_heavy:c_light (heaviest k systems by expected work)
  bool gate = false;           // concurrent fine stage: record / wait evp[2] around the Krylov launches
  cudaEvent_t evc[3] = {};
  cudaEvent_t evcp[2] = {};  // coarse step parts: after the porous solves, after the Navier-Stokes iteration
  long long coarse_n = 0;      // latest coarse time index available
  double coarse_dt = -1.0;
  bool overlap = true;
  int coarse_newton = 1;
  long long ml_built = -1;  // step at which the coarse-box inverses were last built
  int ml_refresh = 1;       // rebuild period (steps)
  double ml_dt = -1.0;  // coarse NS by Newton (same discrete solution as Picard, C11 tolerance); 0 = Picard
  cusolverDnHandle_t sol2 = nullptr;
  double *wpic = nullptr, *wpic2 = nullptr, *ppic = nullptr, *ppic2 = nullptr;
  double* nrm = nullptr;  // 2 doubles
  // composite fine fields at t_n (committed state) and the shadow arrays the running step writes back into;
  // the two sets are swapped when the step commits (lpfem_step: nothing is committed on LPFEM_ENOCONV)
  double* comp[3] = {};
  double* comp_u = nullptr;
  double* comp_p = nullptr;
  double* comp2[3] = {};
  double* comp2_u = nullptr;
  double* comp2_p = nullptr;
  // time levels (C18): t_{n+1} = t_base + (n + 1 - n_base) dt, (n_base, t_base) = where the current dt took effect
  double t_now = 0.0, t_base = 0.0;
  long long n_base = 0;
  int fault_maxit[2] = {0, 0};  // lpfem_inject_fault: cap of the fine Krylov iterations (0 = none)
  bool pending_ok = true;       // convergence verdict of the step in flight (step_begin .. step_end)
  double pending_t = 0.0;
  double pending_res[2] = {0, 0};
  // Algorithm 1 on T_h at scale (lpfem_opts.algorithm = 1, H > h): Newton iterates of the fine conduit step and the
  // iterate injected into the coarse P2 layout (linearisation point of the preconditioner's coarse-box operators)
  bool alg1k = false;
  double *a1u[2] = {}, *a1p[2] = {}, *a1uH = nullptr;
  bool alg1_ok = true;
  double alg1_gm_ms = 0.0;  // GMRES device time of the Newton iterations of the step in flight
  long long n2p_f = 0, n2c_f = 0, n1c_f = 0, n2p_c = 0, n2c_c = 0, n1c_c = 0;
  double* kmult = nullptr;
  std::vector<double> hkmult;
  void* ref = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[4] = {};
  cudaEvent_t ek[4] = {};
  lpfem_stats stats{};
  std::string err;
  long long nstep = 0;
  double cur_dt = -1.0;
  double schur_c = 1.0;
  double vw = 1.0, pw = 1.0;  // preconditioner scaling weights (velocity levels, pressure Schur approximation)
  // multilevel preconditioner of the fine conduit systems (mlprec.cuh)
  int nl = 0;
  Level Llv[NLMAX];
  Family lvl[NLMAX];
  MLArgs ml{};
  double *part = nullptr, *aci = nullptr, *abuf = nullptr, *lwk = nullptr;
  float* ainv[2] = {nullptr, nullptr};   // row-major coarse-box inverses (fp32), double-buffered (coarse_box_inverses)
  __nv_bfloat16* ainvb[2] = {nullptr, nullptr};  // experiment LPFEM_ML_BF16: the same in bf16
  double* cstab = nullptr;               // reference tables of the conduit assembly (k_cstep_tables)
  int ml_next = 0, ml_busy = 0;          // slot the next fine step uses / slot the enqueued fine step reads
  int warm_order = 2;                    // Krylov initial guess: 1 previous solution, 2 linear extrapolation
  // experiment switches (environment, read once at create)
  struct Knobs {
    bool verbose = false, no_smem_pattern = false, cold_start = false, coarse_full_newton = false;
    bool no_concurrent = false, no_alg1_fastpath = false, no_overlap = false;
    bool pcg_ungated = false;  // experiment: the porous PCG launches without waiting for the GMRES launch
    double reorth2 = 0.1;
    int gj_max = 512;
    double pcg_rr_fac = 1e-10;  // mixed-precision PCG: true-residual replacement when ||r||^2 fell by this factor
  } kn;
  // coarse Navier-Stokes chord iteration: LU of the last factorised Jacobian in `dense`/`piv` (conduit_solve_once)
  bool clu_valid = false, clu_force = false;
  int clu_newton = -1;
  double clu_dt = -1.0;
  double* lwk2 = nullptr;                // cuSOLVER workspace of sol2 (coarse stream)
  int *lpiv2 = nullptr, *linfo2 = nullptr;
  // 3D coarse-box inverses: NSI concurrent cuSOLVER streams (one LU + solve-with-identity per box, round robin)
  static constexpr int NSI = 8;
  int nsi = 0;
  cudaStream_t sinv[NSI] = {};
  cusolverDnHandle_t hinv[NSI] = {};
  double* lwki[NSI] = {};
  int *lpivi[NSI] = {}, *linfoi[NSI] = {};
  cudaEvent_t einv[NSI + 1] = {};
  long long *dpoff = nullptr, *daoff = nullptr;
  std::vector<long long> haoff;
  int *lpiv = nullptr, *linfo = nullptr;
  int llwork = 0;
  std::vector<void*> stencils;
  int* gjperm = nullptr;  // pivot scratch of the batched Gauss-Jordan inversion
  // multilevel preconditioner of the fine porous PCG (same level ratios, scalar P2)
  int nlp = 0;
  Family plv[NLMAX];
  Level Lplv[NLMAX];
  MLArgs mlp{};
  double *aci_p = nullptr, *abuf_p = nullptr;
  int* gjperm_p = nullptr;        // porous: pivot scratch of the batched Gauss-Jordan inversion
  SysDesc* pds3 = nullptr;        // porous coarse-box descriptors, one per (field, box) system
  long long* daoff_p = nullptr;
  std::vector<long long> haoff_p;
  // multi-GPU (world > 1): NCCL communicator or local group, halo plan, exchange buffers
  ncclComm_t comm = nullptr;
  std::vector<PeerX> peers;
  std::vector<int> rank_of_pos;  // placement of the subdomain positions (halo.h, LPT)
  HaloPlan plan_p, plan_c2, plan_c1;
  std::vector<int*> own_p, own_c2, own_c1;  // device copies of every rank's owned lists (gather to root)
  double* gbuf = nullptr;  // gather buffer
  long long gbuf_n = 0;
  int* dok = nullptr;            // NCCL: convergence verdict, min-reduced over the ranks
  cudaEvent_t ev_pack = nullptr; // local transport: this rank's send buffers are packed
  cudaEvent_t ev_xdone = nullptr;  // local transport: this rank's copies out of its peers' buffers are done
  std::string group_key;         // local transport: registry key (dist.nccl_id bytes)
  // coarse Navier-Stokes: dense LU on the device (cuSOLVER), Step 1 dependency (C11)
  cusolverDnHandle_t sol = nullptr;
  double *dense = nullptr, *dwork = nullptr;
  int *piv = nullptr, *dinfo = nullptr;
  int lwork = 0;
};

namespace {

void setup_multi(lpfem_ctx* c);
RegionGrid region_grid(const lpfem_ctx* c, int reg);

// ------------------------------------------------------------------------------------ host setup
void upload_tables() {
  // __constant__ tables live per device: upload once per device of this process
  static std::mutex mu;
  static bool done_dev[256] = {};
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 256) throw Err(LPFEM_EINVAL, "device index");
  bool& done = done_dev[dev];
  if (done) return;
  KuhnTables kt[4];
  for (int d = 1; d <= 3; ++d) build_kuhn(d, kt[d]);
  CK(cpysym(c_kt, kt, sizeof(kt)));
  // neighbour offsets per parity class, from the simplices around an interior reference node
  static signed char nb[4][8][72][3], nb1[4][8][32][3];
  static int nbn[4][8], nb1n[4][8];
  std::memset(nb, 0, sizeof(nb));
  std::memset(nb1, 0, sizeof(nb1));
  std::memset(nbn, 0, sizeof(nbn));
  std::memset(nb1n, 0, sizeof(nb1n));
  for (int d = 2; d <= 3; ++d) {
    const KuhnTables& T = kt[d];
    const int nt = nt_of(d), N = n2_of(d);
    for (int k = 0; k < (1 << d); ++k) {
      int l[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a) l[a] = 8 + ((k >> a) & 1);
      std::vector<std::array<int, 3>> p2, p1;
      for (int c2 = 2; c2 <= (d > 2 ? 6 : 2); ++c2)
        for (int c1 = 2; c1 <= 6; ++c1)
          for (int c0 = 2; c0 <= 6; ++c0) {
            int c[3] = {c0, c1, d > 2 ? c2 : 0};
            bool inside = true;
            int code = 0, s = 1;
            for (int a = 0; a < d; ++a, s *= 3) {
              int o = l[a] - 2 * c[a];
              inside = inside && o >= 0 && o <= 2;
              code += o * s;
            }
            if (!inside) continue;
            for (int t = 0; t < nt; ++t) {
              if (T.lookup[t][code] < 0) continue;
              for (int j = 0; j < N; ++j) {
                std::array<int, 3> v = {0, 0, 0};
                for (int a = 0; a < d; ++a) v[a] = 2 * c[a] + T.off[t][j][a] - l[a];
                p2.push_back(v);
                if (j <= d) p1.push_back(v);
              }
            }
          }
      auto key = [](const std::array<int, 3>& v) { return ((v[2] + 4) * 9 + (v[1] + 4)) * 9 + (v[0] + 4); };
      auto srt = [&](std::vector<std::array<int, 3>>& vv) {
        std::sort(vv.begin(), vv.end(), [&](auto& a, auto& b) { return key(a) < key(b); });
        vv.erase(std::unique(vv.begin(), vv.end()), vv.end());
      };
      srt(p2);
      srt(p1);
      if (p2.size() > 72 || p1.size() > 32) throw Err(LPFEM_EINVAL, "neighbour table overflow");
      nbn[d][k] = (int)p2.size();
      nb1n[d][k] = (int)p1.size();
      for (size_t i = 0; i < p2.size(); ++i)
        for (int a = 0; a < 3; ++a) nb[d][k][i][a] = (signed char)p2[i][a];
      for (size_t i = 0; i < p1.size(); ++i)
        for (int a = 0; a < 3; ++a) nb1[d][k][i][a] = (signed char)p1[i][a];
    }
  }
  CK(cpysym(c_nb, nb, sizeof(nb)));
  CK(cpysym(c_nbn, nbn, sizeof(nbn)));
  CK(cpysym(c_nb1, nb1, sizeof(nb1)));
  CK(cpysym(c_nb1n, nb1n, sizeof(nb1n)));
  done = true;
}

int to_int_checked(double v, lpfem_status code, const char* what) {
  double r = std::round(v);
  if (r < 1 || std::fabs(v - r) > 1e-12 * std::max(1.0, std::fabs(v)))
    throw Err(code, std::string(what) + " is not a positive integer");
  return (int)r;
}

LevelGeom make_level(int D, const double* lo, const double* hi, int region, double step, int R) {
  LevelGeom G{};
  for (int a = 0; a < 3; ++a) {
    G.n[a] = 1;
    G.lo[a] = 0;
    G.hi[a] = 0;
    G.hc[a] = 1;
    G.hg[a] = 1;
  }
  for (int a = 0; a < D; ++a) {
    G.n[a] = to_int_checked((hi[a] - lo[a]) / step, LPFEM_ENOTDIV, "region extent / mesh size");
    G.lo[a] = lo[a];
    G.hi[a] = hi[a];
    G.hc[a] = (hi[a] - lo[a]) / G.n[a];
    G.hg[a] = (hi[a] - lo[a]) / (2 * G.n[a]);
  }
  G.R = R;
  G.region = region;
  G.far_g = region == 0 ? 0 : 2 * G.n[D - 1];
  G.gamma_g = region == 0 ? 2 * G.n[D - 1] : 0;
  return G;
}

inline dim3 grid_rows(int maxrows, int nsys, int bs = 128) { return dim3((maxrows + bs - 1) / bs, nsys); }

template <int D>
void build_pattern(lpfem_ctx* c, Family& F) {
  cudaStream_t st = c->st;
  const int nsys = (int)F.hs.size();
  F.ds = dalloc<SysDesc>(nsys);
  CK(cpya(F.ds, F.hs.data(), nsys * sizeof(SysDesc), cudaMemcpyHostToDevice, st));
  long long* cnt = dalloc<long long>(F.rows + 1);
  CK(cudaMemsetAsync(cnt, 0, (F.rows + 1) * sizeof(long long), st));
  k_pattern_count<D><<<grid_rows(F.maxrows, nsys), 128, 0, st>>>(F.ds, F.kind, cnt);
  CKL();
  F.rowptr = dalloc<long long>(F.rows + 1);
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, F.rowptr, F.rows + 1, st));
  void* dtmp = dalloc<char>(tmp);
  CK(cub::DeviceScan::ExclusiveSum(dtmp, tmp, cnt, F.rowptr, F.rows + 1, st));
  CK(cpya(&F.nnz, F.rowptr + F.rows, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dtmp);
  cudaFree(cnt);
  {
    std::vector<long long> rp(F.rows + 1);
    CK(cpy(rp.data(), F.rowptr, (F.rows + 1) * sizeof(long long), cudaMemcpyDeviceToHost));
    for (auto& S : F.hs) F.sys_nnz.push_back(rp[S.row_off + S.nrows] - rp[S.row_off]);
    F.hrp = std::move(rp);
  }
  F.col = dalloc<int>(F.nnz);
  k_pattern_fill<D><<<grid_rows(F.maxrows, nsys), 128, 0, st>>>(F.ds, F.kind, F.rowptr, F.col);
  CKL();
}

// node-blocked copy of a conduit family's operator (krylov.cuh NBMat): lengths, pointers and columns (once)
template <int D>
void build_nb(lpfem_ctx* c, Family& F) {
  cudaStream_t st = c->st;
  const int ns = (int)F.hs.size();
  const long long ni = F.nb_items;
  F.nbioff = dalloc<long long>(ns);
  CK(cpy(F.nbioff, F.h_ioff.data(), ns * sizeof(long long), cudaMemcpyHostToDevice));
  F.nblen = dalloc<int2>(ni);
  long long* cc = dalloc<long long>(ni + 1);
  long long* vc = dalloc<long long>(ni + 1);
  CK(cudaMemsetAsync(cc, 0, (ni + 1) * sizeof(long long), st));
  CK(cudaMemsetAsync(vc, 0, (ni + 1) * sizeof(long long), st));
  k_nb_len<D><<<grid_rows(F.maxitems, ns), 128, 0, st>>>(F.ds, F.nbioff, F.rowptr, F.col, F.nblen, cc, vc);
  CKL();
  F.nbcptr = dalloc<long long>(ni + 1);
  F.nbvptr = dalloc<long long>(ni + 1);
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cc, F.nbcptr, ni + 1, st));
  void* dtmp = dalloc<char>(tmp);
  CK(cub::DeviceScan::ExclusiveSum(dtmp, tmp, cc, F.nbcptr, ni + 1, st));
  CK(cub::DeviceScan::ExclusiveSum(dtmp, tmp, vc, F.nbvptr, ni + 1, st));
  long long tot[2];
  CK(cpya(&tot[0], F.nbcptr + ni, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cpya(&tot[1], F.nbvptr + ni, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFree(dtmp);
  cudaFree(cc);
  cudaFree(vc);
  if (tot[1] != F.nnz) throw Err(LPFEM_ESTATE, "node-blocked operator: value count differs from the CSR");
  F.nb_ncols = tot[0];
  F.nbcol = dalloc<int>(F.nb_ncols);
  F.nbval = dalloc<double>(F.nnz);
  // fp32 copy of the values for the GMRES's Arnoldi products (krylov.cuh k_gmres); LPFEM_NB_F64=1 (experiment)
  // multiplies with the fp64 values throughout
  if (!getenv("LPFEM_NB_F64")) F.nbval32 = dalloc<float>(F.nnz);
  k_nb_cols<D><<<grid_rows(F.maxitems, ns), 128, 0, st>>>(F.ds, F.nbioff, F.rowptr, F.col, F.nblen, F.nbcptr, F.nbcol);
  CKL();
  // 16-bit column offsets (2 instead of 4 B per (item, neighbour)): a column lies within a few grid planes of the
  // item's first column in a box's lexicographic numbering.  Experiment (LPFEM_NB_COL16=1): measured slower (cfg4
  // standalone SpMV 2.07 -> 2.47 ms, GMRES 747 -> 839 ms per step: the per-item base load and the adds sit in the
  // dependent column -> gather chain), so the 32-bit columns stay the default
  if (getenv("LPFEM_NB_COL16")) {
    F.nbcol16 = dalloc<unsigned short>(F.nb_ncols);
    F.nbcbase = dalloc<int2>(ni);
    int* dbad = dalloc<int>(1);
    CK(cudaMemsetAsync(dbad, 0, sizeof(int), st));
    k_nb_cols16<D><<<grid_rows(F.maxitems, ns), 128, 0, st>>>(F.ds, F.nbioff, F.nblen, F.nbcptr, F.nbcol, F.nbcol16,
                                                              F.nbcbase, dbad);
    CKL();
    int bad = 0;
    CK(cpya(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(dbad);
    if (bad) {
      cudaFree(F.nbcol16);
      cudaFree(F.nbcbase);
      F.nbcol16 = nullptr;
      F.nbcbase = nullptr;
    }
  }
}

// the warp-per-node conduit assembly keeps a node's rows in shared memory (CStepW<D>::RMAX entries per row)
template <int D>
void check_row_len(const Family& F) {
  long long mx = 0;
  for (size_t i = 0; i + 1 < F.hrp.size(); ++i) mx = std::max(mx, F.hrp[i + 1] - F.hrp[i]);
  if (mx > CStepW<D>::RMAX) throw Err(LPFEM_ESTATE, "conduit row longer than the assembly buffer");
}

void alloc_vectors(lpfem_ctx* c, Family& F, bool level_family = false) {
  const long long nv = F.kind == 0 ? 3 * F.rows : F.rows;
  F.base = dalloc<double>(nv);
  F.z = dalloc<double>(nv);
  F.lag = dalloc<double>(nv);
  F.qf = dalloc<double>(nv);
  F.aux = dalloc<double>(F.rows);
  F.rhs = dalloc<double>(nv);
  F.x = dalloc<double>(nv);
  F.r = dalloc<double>(nv);
  F.p = dalloc<double>(nv);
  CK(cudaMemsetAsync(F.x, 0, nv * sizeof(double), c->st));
  if (!level_family && F.level == 1) {  // Krylov warm start: the solution one step before x
    F.xp = dalloc<double>(nv);
    CK(cudaMemsetAsync(F.xp, 0, nv * sizeof(double), c->st));
  }
  if (F.kind == 0) {
    F.val = dalloc<double>(3 * F.nnz);
    F.diag = dalloc<double>(nv);
    F.isq = dalloc<double>(nv);
    F.wn = dalloc<double>(nv);
    F.q = dalloc<double>(nv);
  } else {
    F.aconst = dalloc<double>(F.nnz);
    F.aout = dalloc<double>(F.nnz);
    F.scale = dalloc<double>(F.rows);
    F.mask = dalloc<double>(F.rows);
    F.W = dalloc<double>(F.rows);
    F.q = dalloc<double>(F.rows);
    if (!level_family) F.V = dalloc<double>((size_t)(GM + 1) * F.rows);
  }
  if (level_family) return;
  if (F.level == 1 && c->opts.lag_mode == LPFEM_LAG_SUBDOMAIN) {
    F.ecorr = dalloc<double>(nv);
    F.ecorr2 = dalloc<double>(nv);
    CK(cudaMemsetAsync(F.ecorr, 0, nv * sizeof(double), c->st));
    CK(cudaMemsetAsync(F.ecorr2, 0, nv * sizeof(double), c->st));
  }
  // Krylov system list
  const int nsub = (int)F.hs.size();
  if (F.kind == 0) {
    for (int f = 0; f < 3; ++f)
      for (int s = 0; s < nsub; ++s) {
        KSys k{};
        k.row_off = f * F.rows + F.hs[s].row_off;
        k.prow_off = F.hs[s].row_off;
        k.val_off = f * F.nnz;
        k.nrows = F.hs[s].nrows;
        F.hk.push_back(k);
      }
  } else {
    long long io = 0;
    for (int s = 0; s < nsub; ++s) {
      KSys k{};
      k.row_off = F.hs[s].row_off;
      k.prow_off = F.hs[s].row_off;
      k.val_off = 0;
      k.nrows = F.hs[s].nrows;
      k.item_off = io;
      k.n2 = F.hs[s].n2;
      k.n1 = F.hs[s].n1;
      F.h_ioff.push_back(io);
      io += F.hs[s].n2 + F.hs[s].n1;
      F.hk.push_back(k);
    }
    F.nb_items = io;
  }
  F.dk = dalloc<KSys>(F.hk.size());
  CK(cpya(F.dk, F.hk.data(), F.hk.size() * sizeof(KSys), cudaMemcpyHostToDevice, c->st));
  F.dstat = dalloc<KStat>(F.hk.size());
  F.hstat.resize(F.hk.size());
}

// Restriction stencils for ratio q: weights phi_I(x_g) of an interior coarse node I of each parity class at
// the fine half-grid points g = q l + delta (exact rationals, rounded once).
template <int D>
void build_stencil(int q, Stencil& T) {
  std::memset(&T, 0, sizeof(T));
  T.q = q;
  KuhnTables kt;
  build_kuhn(D, kt);
  int n = 0;
  for (int cls = 0; cls < 9; ++cls) {
    if (cls >= (1 << D) && cls != 8) continue;
    T.start[cls] = n;
    int l[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) l[a] = cls == 8 ? 8 : 8 + ((cls >> a) & 1);
    int rng = 2 * q;
    int d[3];
    for (d[2] = (D > 2 ? -rng : 0); d[2] <= (D > 2 ? rng : 0); ++d[2])
      for (d[1] = -rng; d[1] <= rng; ++d[1])
        for (d[0] = -rng; d[0] <= rng; ++d[0]) {
          if (cls == 8 && ((d[0] & 1) || (d[1] & 1) || (d[2] & 1))) continue;
          int g[3] = {0, 0, 0};
          for (int a = 0; a < D; ++a) g[a] = q * l[a] + d[a];
          // coarse simplex containing g: cell, numerators, order (as in the prolongation)
          int cell[3], num[3], ord[3] = {0, 1, 2};
          for (int a = 0; a < D; ++a) {
            cell[a] = g[a] / (2 * q);
            num[a] = g[a] - 2 * q * cell[a];
          }
          std::stable_sort(ord, ord + D, [&](int x, int y) { return num[x] > num[y]; });
          long long lam[4];
          lam[0] = 2 * q - num[ord[0]];
          for (int k = 1; k < D; ++k) lam[k] = num[ord[k - 1]] - num[ord[k]];
          lam[D] = num[ord[D - 1]];
          int V[4][3] = {};
          for (int a = 0; a < D; ++a) V[0][a] = 2 * cell[a];
          for (int k = 1; k <= D; ++k) {
            for (int a = 0; a < D; ++a) V[k][a] = V[k - 1][a];
            V[k][ord[k - 1]] += 2;
          }
          double w = 0.0;
          auto same = [&](const int* P) {
            for (int a = 0; a < D; ++a)
              if (P[a] != l[a]) return false;
            return true;
          };
          if (cls == 8) {
            for (int k = 0; k <= D; ++k)
              if (same(V[k])) w = (double)lam[k] / (2.0 * q);
          } else {
            for (int k = 0; k <= D; ++k)
              if (same(V[k])) w = (double)(lam[k] * (lam[k] - q)) / (2.0 * q * q);
            for (int a = 0; a <= D; ++a)
              for (int b = a + 1; b <= D; ++b) {
                int E[3];
                for (int e = 0; e < D; ++e) E[e] = (V[a][e] + V[b][e]) / 2;
                if (same(E)) w = (double)(2 * lam[a] * lam[b]) / (2.0 * q * q);
              }
          }
          if (w != 0.0) {
            if (n >= STMAX) throw Err(LPFEM_EINVAL, "restriction stencil table overflow");
            for (int a = 0; a < 3; ++a) T.off[n][a] = (signed char)(a < D ? d[a] : 0);
            T.w[n] = w;
            ++n;
          }
        }
    T.len[cls] = n - T.start[cls];
  }
}

// one system = the whole region on the coarse level
SysDesc whole_region(int D, const LevelGeom& G, int kind) {
  SysDesc S{};
  for (int a = 0; a < 3; ++a) {
    S.c0[a] = 0;
    S.nc[a] = a < D ? G.n[a] : 0;
    S.np[a] = a < D ? 2 * G.n[a] + 1 : 1;
  }
  S.n2 = 1;
  S.n1 = 1;
  for (int a = 0; a < D; ++a) {
    S.n2 *= S.np[a];
    S.n1 *= S.nc[a] + 1;
  }
  S.nrows = kind == 0 ? S.n2 : D * S.n2 + S.n1;
  S.has_gamma = 1;
  S.level = 0;
  return S;
}

void finish_family(int D, Family& F) {
  long long off = 0;
  F.maxrows = 0;
  F.maxitems = 0;
  for (auto& S : F.hs) {
    S.row_off = off;
    off += S.nrows;
    F.maxrows = std::max(F.maxrows, S.nrows);
    F.maxitems = std::max(F.maxitems, S.n2 + S.n1);
  }
  F.rows = off;
  (void)D;
}

template <int D>
__global__ void k_init_p2(LevelGeom G, ProbData pd, Coef co, int kind, double* o0, double* o1, double* o2,
                          long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int np[3] = {2 * G.n[0] + 1, 2 * G.n[1] + 1, 2 * G.n[2] + 1}, g[3] = {0, 0, 0};
  unlex<D>(i, np, g);
  double x[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) x[a] = __dadd_rn(G.lo[a], __dmul_rn((double)g[a], G.hg[a]));
  double v[3];
  if (kind == 0) {
    porous_values<D>(pd, x, 0.0, v);
  } else {
    // initial velocity I_h u_0: the injection problems start from rest (C16), the inflow acts from t_1 on
    velocity_values<D>(pd, x, 0.0, false, v);
  }
  o0[i] = v[0];
  o1[i] = v[1];
  if (o2) o2[i] = v[2];
}

template <int D>
__global__ void k_init_p1(LevelGeom G, ProbData pd, Coef co, double* o, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int nv[3] = {G.n[0] + 1, G.n[1] + 1, G.n[2] + 1}, v[3] = {0, 0, 0};
  unlex<D>(i, nv, v);
  double x[3] = {0, 0, 0};
  for (int a = 0; a < D; ++a) x[a] = __dadd_rn(G.lo[a], __dmul_rn((double)(2 * v[a]), G.hg[a]));
  o[i] = pressure_value<D>(pd, co, x, 0.0);
}

// dense column-major copy of the single coarse saddle system A' (fixed rows/columns -> identity)
__global__ void k_csr_to_dense(const long long* __restrict__ rowptr, const int* __restrict__ col,
                               const double* __restrict__ val, const double* __restrict__ s, int n,
                               double* __restrict__ A) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  if (s[r] == 0.0) {
    A[(long long)r * n + r] = 1.0;
    return;
  }
  for (long long q = rowptr[r]; q < rowptr[r + 1]; ++q) A[(long long)col[q] * n + r] = val[q];
}

__global__ void k_sub(const double* a, const double* b, double* o, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) o[i] = a[i] - b[i];
}

// ||u - w||^2 and ||u||^2 over n entries (single block, fixed order)
__global__ void k_picard_norms(const double* u, const double* w, long long n, double* out) {
  __shared__ double s0[32], s1[32];
  double a = 0.0, b = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = u[i] - w[i];
    a += d * d;
    b += u[i] * u[i];
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) {
    s0[threadIdx.x >> 5] = a;
    s1[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x0 = 0, x1 = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      x0 += s0[k];
      x1 += s1[k];
    }
    out[0] = x0;
    out[1] = x1;
  }
}

template <class Kern, class... Args>
void launch_cluster_sm(Kern k, int nsys, int CL, int NT, size_t smem, cudaStream_t st, const Args&... a) {
  if (nsys == 0) return;
  if (CL > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  if (smem > 0) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsys * CL);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, a...));
  ++tl_launches;
}

// Clusters of a Krylov launch wait on one another only inside a cluster, but the kernel ends with its slowest
// system: every system's cluster must be resident at once, or the late ones run in a second wave (measured
// cfg1: 16 clusters of 8 x 1024-thread CTAs -> one wave does not fit the GPCs, 21 ms instead of 13 ms).
// Returns the largest cluster size <= CLmax whose clusters all fit (any size, not only powers of two: the GPCs
// of a B200 are not all the same size), by the occupancy API.
template <class Kern>
int resident_cluster(Kern k, int nsys, int CLmax, int NT, size_t smem, bool verbose = false) {
  for (int CL = CLmax; CL > 1; --CL) {
    if (CL > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (smem > 0) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsys * CL);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (verbose) fprintf(stderr, "[lpfem] cluster %d: %d systems, %d resident clusters\n", CL, nsys, ncl);
    if (ncl >= nsys) return CL;
  }
  return 1;
}

template <class Kern, class... Args>
void launch_cluster(Kern k, int nsys, int CL, int NT, cudaStream_t st, const Args&... a) {
  launch_cluster_sm(k, nsys, CL, NT, 0, st, a...);
}

// Dynamic shared memory for the CTA patterns staged by the Krylov kernels (krylov.cuh stage_pattern): the
// largest (row offsets + column indices) of any CTA's row block, or 0 when one does not fit next to the
// kernel's static shared memory (the kernels then read the pattern from global memory).
template <class Kern>
size_t pattern_smem(Kern k, const Family& F, int CL, size_t front = 0, bool disabled = false) {
  if (disabled || F.hrp.empty()) return 0;
  cudaFuncAttributes at;
  CK(cudaFuncGetAttributes(&at, k));
  const long long budget = 227LL * 1024 - (long long)at.sharedSizeBytes - (long long)front - 1024;
  long long need = 0;
  for (const KSys& K : F.hk) {
    const int chunk = (K.nrows + CL - 1) / CL;
    for (int cr = 0; cr < CL; ++cr) {
      const int r0 = std::min(K.nrows, cr * chunk), r1 = std::min(K.nrows, r0 + chunk);
      const long long nq = F.hrp[K.prow_off + r1] - F.hrp[K.prow_off + r0];
      need = std::max(need, 4LL * (((r1 - r0) + 4) & ~3) + 4 * nq);
    }
  }
  return need <= budget ? (size_t)need : 0;
}


template <int D>
PorousCoefs porous_coefs(const lpfem_ctx* c, double dt) {
  PorousCoefs pc{};
  const Coef& co = c->co;
  const double gFf = co.sigma_star * co.k[1] / co.mu, gfm = co.sigma * co.k[0] / co.mu;
  for (int f = 0; f < 3; ++f) {
    pc.c[f] = co.phiC[f] / dt;
    pc.kappa[f] = co.k[f] / co.mu;
  }
  pc.gamma[2] = gFf;
  pc.gamma[1] = gfm + gFf;
  pc.gamma[0] = gfm;
  pc.gFf = gFf;
  pc.gfm = gfm;
  return pc;
}

template <int D>
ConduitCoefs conduit_coefs(const lpfem_ctx* c, double dt, double hmin) {
  ConduitCoefs cc{};
  cc.eta = c->co.eta;
  cc.nu = c->co.nu;
  cc.alpha = c->co.alpha;
  cc.rho = c->co.rho;
  cc.mu = c->co.mu;
  cc.kF = c->co.k[2];
  cc.dt = dt;
  cc.schur_w = c->pw * (c->co.nu + hmin * hmin / (c->schur_c * dt));
  cc.vel_w = c->vw;
  return cc;
}

template <int D>
const RefT<D>* refp(const lpfem_ctx* c) {
  return (const RefT<D>*)c->ref;
}

int nHv(const lpfem_ctx* c, int a) { return c->nc_p[a]; }

template <int D>
void conduit_const(lpfem_ctx* c, Family& C, const Level& L, double dt) {
  const int nc = (int)C.hs.size();
  if (!nc) return;
  cudaStream_t st = c->st;
  double hmin = 1e300;
  for (int a = 0; a < D; ++a) hmin = std::min(hmin, L.G.hc[a]);
  const ConduitCoefs cc = conduit_coefs<D>(c, dt, hmin);
  k_conduit_const<D><<<grid_rows(C.maxrows, nc), 128, 0, st>>>(C.ds, L, cc, c->kmult, c->nc_p[0], c->nc_p[1],
                                                                c->nc_p[2], refp<D>(c), C.rowptr, C.col, C.aconst);
  CKL();
  k_conduit_scale<D><<<grid_rows(C.maxrows, nc), 128, 0, st>>>(C.ds, L, cc, C.rowptr, C.col, C.aconst, C.scale);
  CKL();
  k_mask_from_scale<<<(unsigned)((C.rows + 255) / 256), 256, 0, st>>>(C.scale, C.mask, C.rows);
  CKL();
}

// porous multilevel preconditioner: level diagonals and the coarse-box inverses (the porous operators are
// time-invariant for fixed dt, so this runs once per dt)
template <int D>
void porous_levels(lpfem_ctx* c, double dt) {
  cudaStream_t st = c->st;
  const PorousCoefs pc = porous_coefs<D>(c, dt);
  for (int l = 0; l < c->nlp; ++l) {
    Family& F = c->plv[l];
    const int ns = (int)F.hs.size();
    k_porous_assemble<D><<<grid_rows(F.maxrows, ns), 128, 0, st>>>(F.ds, c->Lplv[l], pc, c->kmult, c->nc_p[0],
                                                                    c->nc_p[1], c->nc_p[2], refp<D>(c), F.rowptr,
                                                                    F.col, F.val, F.nnz, F.diag, F.rows);
    CKL();
    k_porous_invdiag<D><<<grid_rows(F.maxrows, ns), 128, 0, st>>>(F.ds, c->Lplv[l], F.diag, F.dinv, F.wn, F.rows);
    CKL();
  }
  Family& F = c->plv[c->nlp - 1];
  const int ns = (int)F.hs.size();
  const long long tot = c->haoff_p.back();
  CK(cudaMemsetAsync(c->abuf_p, 0, tot * sizeof(double), st));
  k_dense_porous<<<dim3((F.maxrows + 127) / 128, 3 * ns), 128, 0, st>>>(F.ds, ns, F.rowptr, F.col, F.val, F.nnz, F.wn,
                                                                      F.rows, c->daoff_p, c->abuf_p);
  CKL();
  int nmax = 1;
  for (auto& S2 : F.hs) nmax = std::max(nmax, S2.nrows);
  if (nmax <= c->kn.gj_max) {
    // one batched in-place Gauss-Jordan launch for all (field, box) systems instead of 2 x 3 x boxes cuSOLVER
    // calls; the column-major inverse in abuf_p, its masked row-major copy in aci_p
    k_gj_inverse<1024><<<3 * ns, 1024, 2 * (size_t)nmax * sizeof(double), st>>>(c->pds3, c->daoff_p, c->abuf_p,
                                                                                c->gjperm_p);
    CKL();
    k_inv_rowmajor_porous<<<dim3(F.maxrows, 3 * ns), 128, 0, st>>>(F.ds, ns, F.wn, F.rows, c->daoff_p, c->abuf_p,
                                                                   c->aci_p);
    CKL();
    c->mlp.aci = c->aci_p;
    return;
  }
  c->mlp.aci = c->abuf_p;
  k_set_identity_n<<<dim3(F.maxrows, 3 * ns), 128, 0, st>>>(F.ds, ns, c->daoff_p, c->aci_p);
  CKL();
  for (int sid = 0; sid < 3 * ns; ++sid) {
    const int n = F.hs[sid % ns].nrows;
    double* As = c->abuf_p + c->haoff_p[sid];
    double* Bs = c->aci_p + c->haoff_p[sid];
    if (cusolverDnDgetrf(c->sol, n, n, As, n, c->lwk, c->lpiv, c->linfo) != CUSOLVER_STATUS_SUCCESS)
      throw Err(LPFEM_ECUDA, "cusolverDnDgetrf (porous coarse box)");
    if (cusolverDnDgetrs(c->sol, CUBLAS_OP_N, n, n, As, n, c->lpiv, Bs, n, c->linfo) != CUSOLVER_STATUS_SUCCESS)
      throw Err(LPFEM_ECUDA, "cusolverDnDgetrs (porous coarse box)");
  }
  k_inv_rowmajor_porous<<<dim3(F.maxrows, 3 * ns), 128, 0, st>>>(F.ds, ns, F.wn, F.rows, c->daoff_p, c->aci_p,
                                                                 c->abuf_p);
  CKL();
}

template <int D>
void assemble_dt(lpfem_ctx* c, double dt) {
  cudaStream_t st = c->st;
  const PorousCoefs pc = porous_coefs<D>(c, dt);
  for (int lev = 0; lev < 2; ++lev) {
    Family& P = c->fam[lev][0];
    const int ns = (int)P.hs.size();
    if (ns) {
      k_porous_assemble<D><<<grid_rows(P.maxrows, ns), 128, 0, st>>>(
          P.ds, c->Lp[lev], pc, c->kmult, c->nc_p[0], c->nc_p[1], c->nc_p[2], refp<D>(c), P.rowptr, P.col, P.val,
          P.nnz, P.diag, P.rows);
      CKL();
      if (lev == 1 && c->nlp > 0) {
        // multilevel PCG: masked unscaled operator; isq := 0/1 mask, dinv = 1/diag for the fine Jacobi part
        k_porous_invdiag<D><<<grid_rows(P.maxrows, ns), 128, 0, st>>>(P.ds, c->Lp[lev], P.diag, P.dinv, P.isq, P.rows);
      } else {
        k_porous_isq<D><<<grid_rows(P.maxrows, ns), 128, 0, st>>>(P.ds, c->Lp[lev], P.diag, P.isq, P.rows);
      }
      CKL();
      k_porous_scale<D><<<grid_rows(P.maxrows, ns), 128, 0, st>>>(P.ds, P.rowptr, P.col, P.val, P.nnz, P.isq,
                                                                   P.rows);
      CKL();
      if (P.val32) {
        k_round_f32<<<(unsigned)std::min<long long>((3 * P.nnz + 255) / 256, 148 * 16), 256, 0, st>>>(P.val, P.val32,
                                                                                                     3 * P.nnz);
        CKL();
      }
    }
    conduit_const<D>(c, c->fam[lev][1], c->Lc[lev], dt);
  }
  for (int l = 0; l < c->nl; ++l) conduit_const<D>(c, c->lvl[l], c->Llv[l], dt);
  if (c->nlp > 0) porous_levels<D>(c, dt);
  c->cur_dt = dt;
}

template <int D>
void solve_porous(lpfem_ctx* c, Family& P) {
  KArgs a{};
  a.sys = P.dk;
  a.rowptr = P.rowptr;
  a.col = P.col;
  a.val = P.val;
  a.val32 = P.val32;
  a.rr_fac = c->kn.pcg_rr_fac;
  a.b = P.rhs;
  a.w = P.wn;
  a.x = P.x;
  a.r = P.r;
  a.p = P.p;
  a.q = P.q;
  a.rows_total = 3 * P.rows;
  a.rtol = c->opts.krylov_rtol;
  a.maxit = (P.level == 1 && c->fault_maxit[0] > 0) ? c->fault_maxit[0] : c->opts.max_iter;
  a.stat = P.dstat;
  // warm start from the previous step's corrections (fine ML-PCG): measured fewer iterations, same test (C19)
  a.warm = (P.level == 1 && c->nlp > 0 && !c->kn.cold_start) ? std::min(P.solved, c->warm_order) : 0;
  a.xp = a.warm > 0 ? P.xp : nullptr;
  a.order = P.level == 1 ? P.dorder : nullptr;
  P.solved = std::min(P.solved + 1, 2);
  const int ns = (int)P.hk.size();
  auto go_ml = [&](auto k) {
    if (!P.cluster_checked && !P.bandwidth_bound) {
      P.cluster = resident_cluster(k, P.nsys_rule, P.cluster, 1024, pattern_smem(k, P, P.cluster, 0, c->kn.no_smem_pattern), c->kn.verbose);
      P.cluster_checked = true;
    }
    const size_t sm = pattern_smem(k, P, P.cluster, 0, c->kn.no_smem_pattern);
    a.smem_cols = sm > 0;
    launch_cluster_sm(k, ns, P.cluster, 1024, sm, c->st, a, c->mlp, P.zv);
  };
  auto go = [&](auto k) {
    if (!P.cluster_checked && !P.bandwidth_bound) {
      P.cluster = resident_cluster(k, P.nsys_rule, P.cluster, 1024, pattern_smem(k, P, P.cluster, 0, c->kn.no_smem_pattern), c->kn.verbose);
      P.cluster_checked = true;
    }
    const size_t sm = pattern_smem(k, P, P.cluster, 0, c->kn.no_smem_pattern);
    a.smem_cols = sm > 0;
    launch_cluster_sm(k, ns, P.cluster, 1024, sm, c->st, a);
  };
  if (P.level == 1 && c->nlp > 0) {
    if (D == 2)
      go_ml(k_pcg_ml<1024, 4, 2>);
    else
      go_ml(k_pcg_ml<1024, 8, 3>);
  } else if (D == 2) {
    go(k_cg<1024, 4>);
  } else {
    go(k_cg<1024, 8>);
  }
}

template <int D>
void solve_conduit(lpfem_ctx* c, Family& C) {
  KArgs a{};
  a.sys = C.dk;
  a.rowptr = C.rowptr;
  a.col = C.col;
  a.val = C.aout;
  a.val32 = C.aout32;
  a.b = C.rhs;
  a.x = C.x;
  a.r = C.r;
  a.p = C.W;
  a.V = C.V;
  a.rows_total = C.rows;
  // Algorithm 1's Newton solves are in full-field form (zero base): the pressure's accuracy is the residual
  // tolerance times the saddle point's conditioning, so they run to rtol / 10 (C19 still holds)
  a.rtol = (C.level == 1 && c->alg1k) ? 0.1 * c->opts.krylov_rtol : c->opts.krylov_rtol;
  a.maxit = (C.level == 1 && c->fault_maxit[1] > 0) ? c->fault_maxit[1] : c->opts.max_iter;
  a.stat = C.dstat;
  a.q = C.q;
  // Algorithm 1 on T_h: the unknown is the full field (zero base) and every Newton solve starts from the previous
  // solution (the last iterate; at a step's first iteration u_h^n) without extrapolation
  a.warm = (C.level == 1 && !c->kn.cold_start) ? (c->alg1k ? std::min(C.solved, 1) : std::min(C.solved, c->warm_order)) : 0;
  a.xp = a.warm > 0 ? C.xp : nullptr;
  a.order = C.level == 1 ? C.dorder : nullptr;
  if (C.nbval) {
    a.nb = NBMat{C.nbval, C.nbval32, C.nbcol, C.nbvptr, C.nbcptr, C.nblen, nullptr, nullptr};
  }
  C.solved = std::min(C.solved + 1, 2);
  // reorthogonalise only on severe cancellation (||w'|| < 0.316 ||w||); measured: the Kahan-Parlett 1/sqrt(2)
  // threshold reorthogonalised almost every iteration for identical iteration counts (cfg1-3), +20% GMRES time
  a.reorth2 = c->kn.reorth2;
#ifdef LPFEM_PHASE_TIMERS
  static long long* ph = nullptr;
  const int nsys_ph = (int)C.hk.size();
  if (!ph) ph = dalloc<long long>(16 * 4096);
  CK(cudaMemsetAsync(ph, 0, 16 * nsys_ph * sizeof(long long), c->st));
  a.phase = ph;
  c->ml.phase = ph;
#endif
  const bool pc = C.level == 1 && c->nl > 0;

  const size_t hb = gmres_h_bytes(GM);
  auto go = [&](auto k) {
    if (!C.cluster_checked && !C.bandwidth_bound) {
      C.cluster = resident_cluster(k, C.nsys_rule, C.cluster, NTG, hb + pattern_smem(k, C, C.cluster, hb, c->kn.no_smem_pattern || C.nbval), c->kn.verbose);
      C.cluster_checked = true;
    }
    const size_t sm = pattern_smem(k, C, C.cluster, hb, c->kn.no_smem_pattern || C.nbval);
    a.smem_cols = sm > 0;
    const int nsys = (int)C.hk.size();
    if (c->st4 && C.level == 1 && C.nbval && a.order && c->gm_split[0] < nsys) {
      // experiment: the heaviest systems (launch order = expected work) in one launch with larger clusters, the
      // rest beside it on st4 with smaller ones, so that all clusters fit one wave
      const int kh = c->gm_split[0];
      KArgs al = a;
      al.order = a.order + kh;
      CK(cudaEventRecord(c->evs[0], c->st));
      CK(cudaStreamWaitEvent(c->st4, c->evs[0], 0));
      launch_cluster_sm(k, kh, c->gm_split[1], NTG, hb, c->st, a, c->ml);
      launch_cluster_sm(k, nsys - kh, c->gm_split[2], NTG, hb, c->st4, al, c->ml);
      CK(cudaEventRecord(c->evs[1], c->st4));
      CK(cudaStreamWaitEvent(c->st, c->evs[1], 0));
      return;
    }
    launch_cluster_sm(k, nsys, C.cluster, NTG, hb + sm, c->st, a, c->ml);
  };
  if (pc) {
    if (D == 2)
      go(k_gmres<NTG, TPR2, GM, 2, true>);
    else
      go(k_gmres<NTG, TPR3, GM, 3, true>);
  } else {
    if (D == 2)
      go(k_gmres<NTG, TPR2, GM, 2, false>);
    else
      go(k_gmres<NTG, TPR3, GM, 3, false>);
  }
#ifdef LPFEM_PHASE_TIMERS
  if (C.level == 1) {
    std::vector<long long> h(16 * nsys_ph);
    std::vector<KStat> ks(nsys_ph);
    CK(cpya(h.data(), ph, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, c->st));
    CK(cpya(ks.data(), C.dstat, ks.size() * sizeof(KStat), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    int worst = 0;
    for (int i = 0; i < nsys_ph; ++i)
      if (ks[i].iters > ks[worst].iters) worst = i;
    fprintf(stderr, "[phases] per system (iters, rows, in-loop ms):");
    for (int i = 0; i < nsys_ph; ++i) {
      long long tot = 0;
      for (int k = 0; k < 7; ++k) tot += h[16 * i + k];
      fprintf(stderr, " %d:(%d,%d,%.2f)", i, ks[i].iters, C.hk[i].nrows, tot / 1965.0 / 1000.0);
    }
    fprintf(stderr, "\n");
    fprintf(stderr, "[phases] system %d iters %d, us per iteration:", worst, ks[worst].iters);
    const char* nm[7] = {"sync/V", "prec", "spmv", "cgs1", "cgs2", "cgs3", "norm+givens"};
    for (int k = 0; k < 7; ++k) fprintf(stderr, " %s %.2f", nm[k], h[16 * worst + k] / 1965.0 / std::max(1, ks[worst].iters));
    fprintf(stderr, " | prec sub (restrict/sync per level, coarse, prolong+final):");
    for (int k = 8; k < 16; ++k) fprintf(stderr, " %.2f", h[16 * worst + k] / 1965.0 / std::max(1, ks[worst].iters));
    fprintf(stderr, "\n");
  }
#endif
}

// Cluster sizes of the fine Krylov launches, decided before the first fine stage: the conduit GMRES first (all its
// clusters resident), then the porous PCG, which runs concurrently on st3, gets the SMs the conduit leaves free.
// returns whether the porous and conduit stages run concurrently: not with conduit clusters of more than 8 CTAs
// (cfg3: 16), whose placement the PCG's CTAs fragment so that a GMRES cluster waits for the PCG to end (measured
// cfg3 GMRES 76 -> 105 ms concurrent)
template <int D>
bool decide_fine_clusters(lpfem_ctx* c, bool concurrent) {
  Family& C = c->fam[1][1];
  Family& P = c->fam[1][0];
  if (!C.hk.empty() && !C.cluster_checked && !C.bandwidth_bound) {
    const size_t hb = gmres_h_bytes(GM);
    auto chk = [&](auto k) {
      C.cluster = resident_cluster(k, C.nsys_rule, C.cluster, NTG, hb + pattern_smem(k, C, C.cluster, hb, c->kn.no_smem_pattern || C.nbval), c->kn.verbose);
      C.cluster_checked = true;
    };
    const bool pc = c->nl > 0;
    if (D == 2) {
      if (pc) chk(k_gmres<NTG, TPR2, GM, 2, true>);
      else chk(k_gmres<NTG, TPR2, GM, 2, false>);
    } else {
      if (pc) chk(k_gmres<NTG, TPR3, GM, 3, true>);
      else chk(k_gmres<NTG, TPR3, GM, 3, false>);
    }
  }
  concurrent = concurrent && C.cluster <= 8;
  if (concurrent && !P.hk.empty() && !P.cluster_checked && !P.bandwidth_bound && !C.hk.empty() &&
      !C.bandwidth_bound) {
    const int left = c->nsm - C.nsys_rule * C.cluster;
    P.cluster = std::max(1, std::min(P.cluster, left / P.nsys_rule));
  }
  return concurrent;
}

// LPT launch order of a fine Krylov family: expected work rows x (iterations of the last solve + 1), largest first,
// ties by index (deterministic); uploaded only when it changes.  Scheduling only: every system's arithmetic is the
// same in any order.
void set_order(lpfem_ctx* c, Family& F, bool from_stats) {
  const int n = (int)F.hk.size();
  if (n <= 1 || getenv("LPFEM_NO_ORDER")) return;
  std::vector<double> w(n);
  for (int i = 0; i < n; ++i) w[i] = (double)F.hk[i].nrows * (from_stats ? F.hstat[i].iters + 1.0 : 1.0);
  std::vector<int> o(n);
  for (int i = 0; i < n; ++i) o[i] = i;
  std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return w[a] > w[b]; });
  if (o == F.order) return;
  F.order = o;
  if (!F.dorder) F.dorder = dalloc<int>(n);
  CK(cpya(F.dorder, F.order.data(), n * sizeof(int), cudaMemcpyHostToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));  // F.order may change before the copy would run
}

void fetch_stats(lpfem_ctx* c, Family& F, int kind, bool coarse, double& maxres, bool& ok) {
  if (F.hk.empty()) return;
  CK(cpya(F.hstat.data(), F.dstat, F.hstat.size() * sizeof(KStat), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  long long mx = 0, sum = 0;
  for (auto& s : F.hstat) {
    mx = std::max<long long>(mx, s.iters);
    sum += s.iters;
    maxres = std::max(maxres, s.relres);
    if (!s.converged) ok = false;
  }
  if (coarse) {
    c->stats.coarse_iters[kind] += sum;
  } else {
    c->stats.fine_iters[kind] += sum;
    c->stats.fine_max_iters[kind] = mx;
    // algorithmic bytes: SpMV 12 B/nnz + 32 B/row per pass (node-blocked conduit operator:
    // 8 B/nnz + 4 B per (item, neighbour) column + 24 B per item + 16 B/row); CG vector work 64 B/row per
    // iteration; GMRES 48 B/row per iteration + 16 B/row per basis vector per Gram-Schmidt.
    const int nsub = (int)F.hs.size();
    double bytes = 0.0;
    for (size_t i = 0; i < F.hstat.size(); ++i) {
      const int s = (int)(i % nsub);
      const double rows = F.hk[i].nrows, nz = (double)F.sys_nnz[s];
      const KStat& k = F.hstat[i];
      if (F.nbval) {
        const double items = F.hk[i].n2 + F.hk[i].n1;
        const double ncol = (double)F.nb_ncols * (nz / (double)F.nnz);  // the system's share of the columns
        // the Arnoldi products (one per iteration) read the fp32 values when there is an fp32 copy; the residual
        // checks (warm start, every restart) the fp64 values
        const double vbi = F.nbval32 ? 4.0 : 8.0;
        // (columns: 2 B offsets + 8 B of bases per item with the 16-bit columns, else 4 B)
        const double cb = F.nbcol16 ? 2.0 * ncol + 8.0 * items : 4.0 * ncol;
        bytes += k.iters * (vbi * nz + cb + 24.0 * items + 16.0 * rows) +
                 (k.spmv - k.iters) * (8.0 * nz + cb + 24.0 * items + 16.0 * rows);
      } else {
        const double vbi = (F.aout32 || F.val32) ? 8.0 : 12.0;  // (fp32 values in the Arnoldi / CG products)
        bytes += k.iters * (vbi * nz + 32.0 * rows) + (k.spmv - k.iters) * (12.0 * nz + 32.0 * rows);
      }
      // (fp32 Krylov basis in the multilevel-preconditioned GMRES: 4 B per basis entry read or written)
      const double vb = (kind == 1 && c->nl > 0 && F.level == 1 && LPFEM_BASIS_F32) ? 4.0 : 8.0;
      // GMRES per iteration: the product's output W written once and read by both Gram-Schmidt passes (24 B/row),
      // the new basis vector written (vb), and the j+1 basis vectors read by each pass (2 vb per vector)
      bytes += kind == 0 ? 64.0 * rows * k.iters : (24.0 + vb) * rows * k.iters + 2.0 * vb * rows * k.vsum;
      // multilevel preconditioner, once per iteration: the fine vector read by the restriction and by the fine
      // combine, the fine scaling, the result (32 B/row); every level's restricted vector, scaling and correction
      // (~40 B per level row, the transfers' gathers hit the cache); the dense coarse-box inverse (fp32 conduit,
      // fp64 porous: 4 / 8 B per entry)
      const int nl = kind == 0 ? c->nlp : c->nl;
      if (nl > 0) {
        const Family* lv = kind == 0 ? c->plv : c->lvl;
        double lrows = 0.0;
        for (int l = 0; l < nl; ++l) lrows += lv[l].hs[s].nrows;
        const double nL = lv[nl - 1].hs[s].nrows;
        // (the fine vector read twice: 2 vb for the conduit's basis vector input, 16 for the porous residual)
        const double fin = kind == 0 ? 32.0 : 16.0 + 2.0 * vb;
        bytes += k.iters * (fin * rows + 40.0 * lrows + (kind == 0 ? 8.0 : 4.0) * nL * nL);
      }
    }
    c->stats.bytes_krylov[kind] += bytes;
    c->stats.krylov_launches[kind] += 1;
    set_order(c, F, true);
  }
}

// alg1: Algorithm 1 on T_h (lpfem_opts.algorithm = 1): base and lagged state from the fine composite at the same
// level (mode 2 indexing), the Gamma flux from the fine composite velocity (eq. fullypF)
template <int D>
void porous_stage(lpfem_ctx* c, int lev, double t, double* const* cnew, double* const* cold, const double* cu_old_last,
                  double* const* out, bool alg1 = false) {
  Family& P = c->fam[lev][0];
  const int ns = (int)P.hs.size();
  if (!ns) return;
  cudaStream_t st = c->st;
  PorousPrepArgs A{};
  for (int f = 0; f < 3; ++f) {
    A.coarse_new[f] = cnew[f];
    A.coarse_old[f] = cold[f];
    A.comp[f] = c->comp[f];
  }
  A.coarse_u_old = cu_old_last;
  A.ecorr = P.ecorr;
  for (int a = 0; a < 3; ++a) {
    A.nHp[a] = c->nc_p[a];
    A.nHc[a] = c->nc_c[a];
    A.np_glob[a] = 2 * c->Lp[lev].G.n[a] + 1;
  }
  A.Rp = lev == 0 ? 1 : c->R;
  A.conduit_gamma_g = 0;
  A.mode = lev == 0 ? 2 : (c->opts.lag_mode == LPFEM_LAG_SUBDOMAIN ? 1 : 0);
  A.t = t;
  for (int a = 0; a < 3; ++a) A.nHu[a] = A.nHc[a];
  A.Ru = A.Rp;
  if (alg1) {
    A.mode = 2;
    A.zero_base = 1;
    A.Rp = 1;
    A.Ru = 1;
    for (int a = 0; a < 3; ++a) A.nHu[a] = c->nf_c[a];
  }
  k_porous_prep<D><<<grid_rows(P.maxrows, ns), 128, 0, st>>>(P.ds, c->Lp[lev], c->pd, c->co, A, P.base, P.z, P.lag,
                                                              P.qf, P.aux, P.rows);
  CKL();
  const PorousCoefs pc = porous_coefs<D>(c, c->cur_dt);
  k_porous_rhs<D><<<grid_rows(P.maxrows, ns), 128, 0, st>>>(P.ds, c->Lp[lev], pc, c->kmult, c->nc_p[0], c->nc_p[1],
                                                             c->nc_p[2], refp<D>(c), P.z, P.lag, P.qf, P.aux, P.isq,
                                                             P.rhs, P.wn, P.rows);
  CKL();
  if (lev == 1 && c->gate && !c->kn.pcg_ungated) CK(cudaStreamWaitEvent(st, c->evp[2], 0));  // the GMRES clusters are placed first
  if (lev == 1) CK(cudaEventRecord(c->ek[0], st));
  solve_porous<D>(c, P);
  if (lev == 1) CK(cudaEventRecord(c->ek[1], st));
  k_porous_writeback<D><<<grid_rows(P.maxrows, ns), 128, 0, st>>>(
      P.ds, c->Lp[lev], P.z, P.x, P.isq, P.base, P.ecorr2, out[0], out[1], out[2], 2 * c->Lp[lev].G.n[0] + 1,
      2 * c->Lp[lev].G.n[1] + 1, 2 * c->Lp[lev].G.n[2] + 1, P.rows);
  CKL();
}

// per-step conduit operator and right-hand side of a family (conduit.cuh k_conduit_step_w: one warp per node / row)
template <int D>
void conduit_step(cudaStream_t st, Family& F, const Level& L, const ConduitCoefs& cc, int newton, lpfem_ctx* c,
                  const double* colscale, bool fine_main = false) {
  constexpr int WPB = D == 3 ? 16 : 8;  // 3D: 48 KB of tables + 16 x 10 KB of node buffers, one block per SM
  constexpr size_t sm = cstep_smem<D, WPB>();
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_conduit_step_w<D, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  // persistent CTAs (the 48 KB of reference tables are built once per CTA): as many as fit on the GPU at once
  static int ctas = 0;
  if (!ctas) {
    int per_sm = 0, dev = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_conduit_step_w<D, WPB>, WPB * 32, sm));
    ctas = std::max(1, per_sm) * nsm;
  }
  const int nbx = (F.maxitems + WPB - 1) / WPB, nsys = (int)F.hs.size();
  // One CTA per block of WPB nodes; every CTA copies the prebuilt tables (49 KB, L2 hits) instead of building them
  // (the per-CTA build from the reference tensors was 15% of the kernel's instructions).  Persistent CTAs
  // (LPFEM_CSTEP_PERSIST=1, fine family on the main stream; LPFEM_CSTEP_TICKET=1: in-order block tickets) measured
  // 74 -> 52 ms for the kernel, but the next fine step's GMRES got slower (cfg4 746 -> 845 ms per step): the
  // persistent CTAs, each holding an SM's shared memory until the whole launch drains, delay the porous-stream kernels
  // queued behind them, which then occupy the SMs the GMRES clusters are placed on.
  static const int persist = getenv("LPFEM_CSTEP_PERSIST") ? atoi(getenv("LPFEM_CSTEP_PERSIST")) : 0;  // CTAs
  static const bool use_ticket = getenv("LPFEM_CSTEP_TICKET") != nullptr;
  const bool persistent = fine_main && persist > 0;
  if (!c->cstab) {  // the kernel's reference tables, built once (k_cstep_tables), copied by every CTA
    constexpr int tb = cstep_tab_bytes<D>();
    c->cstab = dalloc<double>(tb / 8);
    CK(cudaFuncSetAttribute(k_cstep_tables<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, tb));
    k_cstep_tables<D><<<1, 512, tb, st>>>(refp<D>(c), c->cstab);
    CKL();
    CK(cudaStreamSynchronize(st));  // once: later launches on any stream read the tables
  }
  const int grid = (int)std::min<long long>((long long)nbx * nsys, persistent ? std::min(ctas, persist) : (1LL << 30));
  if (persistent && use_ticket) {
    if (!F.ticket) F.ticket = dalloc<int>(1);
    CK(cudaMemsetAsync(F.ticket, 0, sizeof(int), st));
  }
  k_conduit_step_w<D, WPB><<<grid, WPB * 32, sm, st>>>(F.ds, L, cc, newton, c->kmult, c->nc_p[0], c->nc_p[1], c->nc_p[2],
                                                      refp<D>(c), F.rowptr, F.col, F.aconst, colscale, F.z, F.W, F.lag,
                                                      F.qf, F.aux, F.aout, F.rhs, nbx, nsys,
                                                      persistent && use_ticket ? F.ticket : nullptr, c->cstab);
  CKL();
}

// Newton-linearised operator of every coarse box (level L of the multilevel preconditioner), inverted densely.
// Runs on the coarse stream (st2, cuSOLVER handle sol2) as the last part of coarse_step(n): U^{n+1} is known
// there, so the inverses for fine step n are built while fine step n - 1 still runs.  The row-major result goes
// to ainv[slot], double-buffered against the slot the running fine step reads.
template <int D>
void coarse_box_inverses(lpfem_ctx* c, const double* cu_new, int slot) {
  Family& F = c->lvl[c->nl - 1];
  const Level& L = c->Llv[c->nl - 1];
  const int ns = (int)F.hs.size();
  cudaStream_t st = c->st;
  ConduitPrepArgs A{};
  A.cu_new = cu_new;
  for (int a = 0; a < 3; ++a) {
    A.nHc[a] = c->nc_c[a];
    A.nHp[a] = c->nc_p[a];
    A.np_glob[a] = 2 * L.G.n[a] + 1;
  }
  A.R = L.G.R;
  A.mode = 3;
  k_conduit_prep<D><<<grid_rows(F.maxitems, ns), 128, 0, st>>>(F.ds, L, c->pd, c->co, A, F.base, F.z, F.W, F.lag,
                                                               F.qf, F.aux);
  CKL();
  double hmin = 1e300;
  for (int a = 0; a < D; ++a) hmin = std::min(hmin, L.G.hc[a]);
  const ConduitCoefs cc = conduit_coefs<D>(c, c->cur_dt, hmin);
  conduit_step<D>(st, F, L, cc, 1, c, F.mask);
  const long long tot = c->haoff.back();
  CK(cudaMemsetAsync(c->abuf, 0, tot * sizeof(double), st));
  k_dense_batched<<<grid_rows(F.maxrows, ns), 128, 0, st>>>(F.ds, F.rowptr, F.col, F.aout, F.mask, c->daoff, c->abuf);
  CKL();
  int nmax = 1;
  for (auto& S2 : F.hs) nmax = std::max(nmax, S2.nrows);
  const double* cm = c->aci;  // column-major inverses
  if (nmax <= c->kn.gj_max) {
    // small boxes (2D): batched in-place Gauss-Jordan, one CTA per matrix
    const size_t smem = 2 * (size_t)nmax * sizeof(double);
    k_gj_inverse<1024><<<ns, 1024, smem, st>>>(F.ds, c->daoff, c->abuf, c->gjperm);
    CKL();
    cm = c->abuf;
  } else {
    // large boxes (3D): dense LU per matrix (cuSOLVER), inverse by solving with the identity; the boxes are
    // spread round robin over nsi streams with their own handles and workspaces (one box's LU does not fill the
    // GPU: n = 1.1k-2.3k at cfg4)
    k_set_identity<<<dim3(F.maxrows, ns), 128, 0, st>>>(F.ds, c->daoff, c->aci);
    CKL();
    CK(cudaEventRecord(c->einv[c->nsi], st));
    for (int k = 0; k < c->nsi; ++k) CK(cudaStreamWaitEvent(c->sinv[k], c->einv[c->nsi], 0));
    for (int s2 = 0; s2 < ns; ++s2) {
      const int k = s2 % c->nsi;
      const int n = F.hs[s2].nrows;
      double* As = c->abuf + c->haoff[s2];
      double* Bs = c->aci + c->haoff[s2];
      if (cusolverDnDgetrf(c->hinv[k], n, n, As, n, c->lwki[k], c->lpivi[k], c->linfoi[k]) != CUSOLVER_STATUS_SUCCESS)
        throw Err(LPFEM_ECUDA, "cusolverDnDgetrf (coarse box)");
      if (cusolverDnDgetrs(c->hinv[k], CUBLAS_OP_N, n, n, As, n, c->lpivi[k], Bs, n, c->linfoi[k]) !=
          CUSOLVER_STATUS_SUCCESS)
        throw Err(LPFEM_ECUDA, "cusolverDnDgetrs (coarse box)");
    }
    for (int k = 0; k < c->nsi; ++k) {
      CK(cudaEventRecord(c->einv[k], c->sinv[k]));
      CK(cudaStreamWaitEvent(st, c->einv[k], 0));
    }
  }
  if (c->ainvb[slot])
    k_inv_rowmajor<__nv_bfloat16><<<dim3(F.maxrows, ns), 128, 0, st>>>(F.ds, F.mask, c->daoff, cm, c->ainvb[slot]);
  else
    k_inv_rowmajor<float><<<dim3(F.maxrows, ns), 128, 0, st>>>(F.ds, F.mask, c->daoff, cm, c->ainv[slot]);
  CKL();
}

// alg1: Algorithm 1 on T_h: every input (iterate, lagged velocity, p_F^n on Gamma) is a fine global array indexed
// like the coarse Picard step (mode 2), so the system is the Newton-linearised fine implicit step about the iterate
template <int D>
void conduit_solve_once(lpfem_ctx* c, int lev, double t, const double* cu_new, const double* cp_new,
                        const double* cu_old, const double* cpF_old, double* out_u, double* out_p, bool alg1 = false) {
  Family& C = c->fam[lev][1];
  const int ns = (int)C.hs.size();
  if (!ns) return;
  cudaStream_t st = c->st;
  ConduitPrepArgs A{};
  A.cu_new = cu_new;
  A.cp_new = cp_new;
  A.cu_old = cu_old;
  A.cpF_old = cpF_old;
  A.comp_u = c->comp_u;
  A.ecorr = C.ecorr;
  for (int a = 0; a < 3; ++a) {
    A.nHc[a] = c->nc_c[a];
    A.nHp[a] = c->nc_p[a];
    A.np_glob[a] = 2 * c->Lc[lev].G.n[a] + 1;
  }
  A.R = lev == 0 ? 1 : c->R;
  A.n2_glob = lev == 0 ? c->n2c_c : c->n2c_f;
  A.porous_gamma_g = 2 * c->nc_p[D - 1] * A.R;
  A.mode = lev == 0 ? 2 : (c->opts.lag_mode == LPFEM_LAG_SUBDOMAIN ? 1 : 0);
  A.t = t;
  if (alg1) {
    A.mode = 2;
    A.zero_base = 1;
    A.R = 1;
    for (int a = 0; a < 3; ++a) {
      A.nHc[a] = c->nf_c[a];
      A.nHp[a] = c->nf_p[a];
    }
    A.n2_glob = c->n2c_f;
    A.porous_gamma_g = 2 * c->nf_p[D - 1];
  }
  k_conduit_prep<D><<<grid_rows(C.maxitems, ns), 128, 0, st>>>(C.ds, c->Lc[lev], c->pd, c->co, A, C.base, C.z, C.W,
                                                               C.lag, C.qf, C.aux);
  CKL();
  double hmin = 1e300;
  for (int a = 0; a < D; ++a) hmin = std::min(hmin, c->Lc[lev].G.hc[a]);
  const ConduitCoefs cc = conduit_coefs<D>(c, c->cur_dt, hmin);
  const bool ml = lev == 1 && c->nl > 0;
  if (ml) {  // coarse-box inverses built by coarse_step (coarse stream, one step ahead)
    c->ml_busy = c->ml_next;
    c->ml.acif = c->ainv[c->ml_busy];
    c->ml.acib = c->ainvb[c->ml_busy];
    c->ml.aci = nullptr;
  }
  double* colscale = ml ? C.mask : C.scale;  // ML: masked unscaled operator, M^-1 applied in the kernel
  const int newton = lev == 1 ? 1 : c->coarse_newton;
  conduit_step<D>(st, C, c->Lc[lev], cc, newton, c, colscale, lev == 1 && st == c->st);
  if (C.aout32) {
    k_round_f32<<<(unsigned)std::min<long long>((C.nnz + 255) / 256, 148 * 16), 256, 0, st>>>(C.aout, C.aout32, C.nnz);
    CKL();
  }
  if (C.nbval) {
    k_nb_pack<D><<<grid_rows(C.maxitems * 32, ns), 128, 0, st>>>(C.ds, C.nbioff, C.rowptr, C.aout, C.nbvptr, C.nbval,
                                                                  C.nbval32);
    CKL();
  }
  if (lev == 0) {
    // The system is in correction form around the current iterate z (rhs = b(W) - J(W) z, the nonlinear
    // residual), so any nonsingular matrix gives a convergent fixed-point map near the solution when it is
    // close to J: the chord iteration keeps the LU of the last factorised Jacobian while the iteration
    // contracts (coarse_step decides), and converges to the same discrete solution under the same C11 test.
    const int n = (int)C.rows;
    const bool reuse = c->clu_valid && !c->clu_force && c->clu_newton == newton && c->clu_dt == c->cur_dt;
    if (!reuse) {
      CK(cudaMemsetAsync(c->dense, 0, (size_t)n * n * sizeof(double), st));
      k_csr_to_dense<<<(n + 127) / 128, 128, 0, st>>>(C.rowptr, C.col, C.aout, C.scale, n, c->dense);
      CKL();
      if (cusolverDnDgetrf(c->sol2, n, n, c->dense, n, c->dwork, c->piv, c->dinfo) != CUSOLVER_STATUS_SUCCESS)
        throw Err(LPFEM_ECUDA, "cusolverDnDgetrf");
      c->clu_valid = true;
      c->clu_force = false;
      c->clu_newton = newton;
      c->clu_dt = c->cur_dt;
      c->stats.coarse_factorizations++;
    }
    CK(cpya(C.x, C.rhs, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (cusolverDnDgetrs(c->sol2, CUBLAS_OP_N, n, 1, c->dense, n, c->piv, C.x, n, c->dinfo) != CUSOLVER_STATUS_SUCCESS)
      throw Err(LPFEM_ECUDA, "cusolverDnDgetrs");
    KStat ks{};
    ks.iters = 1;
    ks.converged = 1;
    ks.spmv = 1;
    CK(cpya(C.dstat, &ks, sizeof(KStat), cudaMemcpyHostToDevice, st));
  } else {
    if (lev == 1 && c->gate) CK(cudaEventRecord(c->evp[2], st));
    if (lev == 1) CK(cudaEventRecord(c->ek[2], st));
    solve_conduit<D>(c, C);
    if (lev == 1) CK(cudaEventRecord(c->ek[3], st));
  }
  const int* npg = A.np_glob;
  k_conduit_writeback<D><<<grid_rows(C.maxitems, ns), 128, 0, st>>>(C.ds, c->Lc[lev], C.z, C.x, colscale, C.base,
                                                                    C.ecorr2, out_u, out_p, npg[0], npg[1], npg[2],
                                                                    A.n2_glob);
  CKL();
}

struct StreamSwap {  // route the launches of the shared stage functions to another stream
  lpfem_ctx* c;
  cudaStream_t old;
  StreamSwap(lpfem_ctx* cc, cudaStream_t s) : c(cc), old(cc->st) { cc->st = s; }
  ~StreamSwap() { c->st = old; }
};

// C18: t_{n1} = t_base + (n1 - n_base) dt -- the product form (n1) dt while dt never changed (t_base = 0,
// n_base = 0), and within every later constant-dt segment
double time_at(const lpfem_ctx* c, long long n1, double dt) { return c->t_base + (double)(n1 - c->n_base) * dt; }

// restores the coarse Navier-Stokes solver state when coarse_step leaves, normally or by an exception
struct CoarseGuard {
  lpfem_ctx* c;
  int newton0;
  int nexc;
  explicit CoarseGuard(lpfem_ctx* cc) : c(cc), newton0(cc->coarse_newton), nexc(std::uncaught_exceptions()) {}
  ~CoarseGuard() {
    c->coarse_newton = newton0;
    if (std::uncaught_exceptions() > nexc) c->clu_valid = false;  // the chord LU may be half-built
  }
};

// Step 1: coarse state n -> n+1 (ring slots n % 3 -> (n+1) % 3), Algorithm 1 on T_H, on st2.
template <int D>
void coarse_step(lpfem_ctx* c, long long n, double dt) {
  StreamSwap sw(c, c->st2);
  CoarseGuard guard(c);
  cudaStream_t st = c->st2;
  const int so = (int)(n % 3), sn = (int)((n + 1) % 3);
  const double t = time_at(c, n + 1, dt);  // C18
  bool ok = true;
  CK(cudaEventRecord(c->evc[0], st));
  porous_stage<D>(c, 0, t, c->cst[so], c->cst[so], c->cu[so] + (D - 1) * c->n2c_c, c->cst[sn]);
  {
    double dummy = 0;
    fetch_stats(c, c->fam[0][0], 0, true, dummy, ok);
  }
  CK(cudaEventRecord(c->evcp[0], st));
  const long long nu = (long long)D * c->n2c_c;
  bool pic_ok = false;
  const int newton0 = guard.newton0;
  for (int attempt = 0; attempt < 2 && !pic_ok; ++attempt) {
  if (attempt == 1) c->coarse_newton = 0;  // Newton failed: fall back to Picard from u^n
  CK(cpya(c->wpic, c->cu[so], nu * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cpya(c->ppic, c->cp[so], c->n1c_c * sizeof(double), cudaMemcpyDeviceToDevice, st));
  double du_prev = 0.0;
  if (attempt == 1) c->clu_force = true;
  for (int it = 0; it < c->opts.picard_max; ++it) {
    conduit_solve_once<D>(c, 0, t, c->wpic, c->ppic, c->cu[so], c->cst[so][2], c->wpic2, c->ppic2);
    double dummy = 0;
    fetch_stats(c, c->fam[0][1], 1, true, dummy, ok);
    k_picard_norms<<<1, 1024, 0, st>>>(c->wpic2, c->wpic, nu, c->nrm);
    CKL();
    double hn[2];
    CK(cpya(hn, c->nrm, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::swap(c->wpic, c->wpic2);
    std::swap(c->ppic, c->ppic2);
    c->stats.picard_iters++;
    const double du = std::sqrt(hn[0]), un = std::sqrt(hn[1]);
    if (!(du == du)) break;  // NaN: diverged
    // chord iteration: refactorise at the current iterate when the frozen Jacobian contracts too slowly
    // (or diverges); LPFEM_COARSE_FULL_NEWTON refactorises every iteration (plain Newton / Picard)
    if (c->kn.coarse_full_newton || (it > 0 && du > 0.25 * du_prev) || it >= 12) c->clu_force = true;
    du_prev = du;
    if (du <= c->opts.picard_rtol * un || du <= 1e-14 * std::sqrt((double)nu)) {
      pic_ok = true;
      break;
    }
  }
  }
  c->coarse_newton = newton0;
  if (!pic_ok) throw Err(LPFEM_ENOCONV, "coarse Navier-Stokes iteration did not converge (C11)");
  if (!ok) {
    std::string m = "a coarse Krylov solve did not converge (C19) at n=" + std::to_string(n) + ":";
    for (int k = 0; k < 2; ++k)
      for (auto& st0 : c->fam[0][k].hstat)
        m += " [" + std::to_string(k) + ": it " + std::to_string(st0.iters) + " conv " + std::to_string(st0.converged) +
             " res " + std::to_string(st0.relres) + "]";
    throw Err(LPFEM_ENOCONV, m);
  }
  CK(cpya(c->cu[sn], c->wpic, nu * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cpya(c->cp[sn], c->ppic, c->n1c_c * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cudaEventRecord(c->evcp[1], st));
  // coarse-box inverses of the multilevel preconditioner for fine step n (Newton-linearised at U = P u_H^{n+1};
  // 3D reuses them for ml_refresh steps), into the slot the in-flight fine step does not read
  if (c->nl > 0 && !c->fam[1][1].hs.empty() &&
      (n - c->ml_built >= c->ml_refresh || c->ml_built < 0 || c->ml_dt != dt)) {
    const int slot = 1 - c->ml_busy;
    coarse_box_inverses<D>(c, c->cu[sn], slot);
    c->ml_next = slot;
    c->ml_built = n;
    c->ml_dt = dt;
  }
  CK(cudaEventRecord(c->evc[1], st));
  CK(cudaEventSynchronize(c->evc[1]));
  float ms = 0, m0 = 0, m1 = 0, m2 = 0;
  CK(cudaEventElapsedTime(&ms, c->evc[0], c->evc[1]));
  CK(cudaEventElapsedTime(&m0, c->evc[0], c->evcp[0]));
  CK(cudaEventElapsedTime(&m1, c->evcp[0], c->evcp[1]));
  CK(cudaEventElapsedTime(&m2, c->evcp[1], c->evc[1]));
  c->stats.t_coarse_ms += ms;
  c->stats.t_coarse_part_ms[0] += m0;
  c->stats.t_coarse_part_ms[1] += m1;
  c->stats.t_coarse_part_ms[2] += m2;
  c->coarse_n = n + 1;
  c->coarse_dt = dt;
}

// ---------------------------------------------------------------------------------------------- the step
// lpfem_step = step_begin (coarse n+1 if not ready, fine corrections, write-back into the shadow composite,
// halo pack) -> step_exchange (halo transfer + unpack into the shadow composite) -> step_overlap (coarse n+2
// on the side stream) -> step_verdict (per-rank convergence) -> [reduction over the ranks] -> step_end
// (commit = swap the shadow arrays in, or leave the state at t_n).  lpfem_step_group runs each phase for all
// the contexts of a local group before the next phase.

void halo_pack(lpfem_ctx* c);
void halo_exchange_nccl(lpfem_ctx* c);
void halo_unpack(lpfem_ctx* c);

// coarse P2 node iH <- fine P2 node R gH (nested meshes): injection of D velocity components
template <int D>
__global__ void k_inject_p2(const double* __restrict__ fine, long long n2f, const int* npf, double* __restrict__ crs,
                            long long n2c, int n0, int n1, int n2, int R) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n2c) return;
  const int npc[3] = {2 * n0 + 1, 2 * n1 + 1, 2 * n2 + 1};
  const int npff[3] = {2 * n0 * R + 1, 2 * n1 * R + 1, 2 * n2 * R + 1};
  int g[3] = {0, 0, 0};
  unlex<D>(i, npc, g);
  for (int a = 0; a < D; ++a) g[a] *= R;
  const long long gi = lex<D>(g, npff);
  for (int a = 0; a < D; ++a) crs[a * n2c + i] = fine[a * n2f + gi];
  (void)npf;
}

// Algorithm 1 on T_h at scale, with the batched multilevel Krylov kernels of the fine stage on whole-region
// "subdomains" (grid 1, no overlap; H only sets the preconditioner hierarchy): the porous step (eqs. fullypF-
// fullypm, lagged partners and the Gamma flux of u_h^n) by one preconditioned CG per field; the implicit
// Navier-Stokes step (eq. fullyuc, p_F^n on Gamma) by Newton iterations from u_h^n, each a Newton-linearised Oseen
// solve by preconditioned GMRES (the Algorithm 3 correction operator about the iterate), to the C11 test
// ||du||_2 <= picard_rtol ||u||_2 -- the same discrete solution as Picard (oracle alg1.py).
template <int D>
void alg1_step(lpfem_ctx* c, double t) {
  cudaStream_t st = c->st;
  porous_stage<D>(c, 1, t, c->comp, c->comp, c->comp_u + (D - 1) * c->n2c_f, c->comp2, true);
  const long long nu = (long long)D * c->n2c_f;
  CK(cpya(c->a1u[0], c->comp_u, nu * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cpya(c->a1p[0], c->comp_p, c->n1c_f * sizeof(double), cudaMemcpyDeviceToDevice, st));
  int cur = 0;
  bool conv = false;
  c->alg1_ok = true;
  c->alg1_gm_ms = 0.0;
  for (int it = 0; it < c->opts.picard_max && !conv; ++it) {
    // preconditioner coarse boxes linearised at u_h^n, rebuilt every ml_refresh steps (as for Algorithm 3)
    if (it == 0 && c->nl > 0 && (c->nstep - c->ml_built >= c->ml_refresh || c->ml_built < 0 || c->ml_dt != c->cur_dt)) {
      k_inject_p2<D><<<(unsigned)((c->n2c_c + 255) / 256), 256, 0, st>>>(c->a1u[cur], c->n2c_f, nullptr, c->a1uH, c->n2c_c,
                                                                         c->nc_c[0], c->nc_c[1], c->nc_c[2], c->R);
      CKL();
      coarse_box_inverses<D>(c, c->a1uH, c->ml_next);
      c->ml_built = c->nstep;
      c->ml_dt = c->cur_dt;
    }
    conduit_solve_once<D>(c, 1, t, c->a1u[cur], c->a1p[cur], c->comp_u, c->comp[2], c->a1u[1 - cur], c->a1p[1 - cur],
                          true);
    double dummy = 0;
    bool ok = true;
    fetch_stats(c, c->fam[1][1], 1, false, dummy, ok);
    c->pending_res[1] = std::max(c->pending_res[1], dummy);
    if (!ok) c->alg1_ok = false;
    k_picard_norms<<<1, 1024, 0, st>>>(c->a1u[1 - cur], c->a1u[cur], nu, c->nrm);
    CKL();
    double hn[2];
    CK(cpya(hn, c->nrm, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float mk = 0.0f;
    CK(cudaEventElapsedTime(&mk, c->ek[2], c->ek[3]));
    c->alg1_gm_ms += mk;
    cur = 1 - cur;
    c->stats.picard_iters++;
    const double du = std::sqrt(hn[0]), un = std::sqrt(hn[1]);
    if (!(du == du)) break;
    conv = du <= c->opts.picard_rtol * un || du <= 1e-14 * std::sqrt((double)nu);
  }
  if (!conv) c->alg1_ok = false;
  CK(cpya(c->comp2_u, c->a1u[cur], nu * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CK(cpya(c->comp2_p, c->a1p[cur], c->n1c_f * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

template <int D>
void step_begin(lpfem_ctx* c, double dt) {
  CK(cudaSetDevice(c->dist.device));
  if (dt != c->cur_dt) {
    CK(cudaStreamSynchronize(c->st2));
    assemble_dt<D>(c, dt);  // on st; the coarse stream must see the new operators
    CK(cudaEventRecord(c->ev[3], c->st));
    CK(cudaStreamWaitEvent(c->st2, c->ev[3], 0));
    c->coarse_n = -1;  // a precomputed coarse step used the old dt
    c->t_base = c->t_now;  // C18: the new dt takes effect at the committed state t_n
    c->n_base = c->nstep;
  }
  cudaStream_t st = c->st;
  const long long n = c->nstep;
  const double t = time_at(c, n + 1, dt);  // C18
  c->pending_ok = true;
  c->pending_t = t;
  c->pending_res[0] = c->pending_res[1] = 0.0;
  if (c->alg1k) {  // Algorithm 1 on T_h: no coarse step, no local corrections
    CK(cudaEventRecord(c->ev[1], st));
    decide_fine_clusters<D>(c, false);
    alg1_step<D>(c, t);
    return;
  }
  // ---------------- Step 1: coarse state n+1 (precomputed during the previous step when dt is unchanged; a
  // precomputed step that did not converge left coarse_n behind, so it is recomputed -- and reported -- here)
  if (c->coarse_n != n + 1 || c->coarse_dt != dt) {
    c->coarse_n = n;
    coarse_step<D>(c, n, dt);
  }
  CK(cudaEventRecord(c->evc[2], c->st2));
  CK(cudaStreamWaitEvent(st, c->evc[2], 0));
  const int so = (int)(n % 3), sn = (int)((n + 1) % 3);
  // ---------------- Steps 3-4: fine corrections + write-back into the shadow composite comp2
  CK(cudaEventRecord(c->ev[1], st));
  // the porous and conduit corrections of a step are independent (each reads only coarse data and its own
  // region's lagged composite): the porous stage runs on st3 beside the conduit stage, its PCG gated behind the
  // GMRES launch so that the GMRES clusters are placed first (ungated, the PCG fragmented the GPCs and a GMRES
  // cluster ran in a second wave).  Measured fine stage cfg0/1/2/3/4: 4.9/12.9/172/96/2327 ->
  // 4.5/11.4/150/91/2141 ms.  LPFEM_NO_CONCURRENT=1 serialises.
  const bool alg1 = c->R == 1 && !c->kn.no_alg1_fastpath;
  bool conc = c->st3 && !c->kn.no_concurrent;
  if (!alg1) conc = decide_fine_clusters<D>(c, conc);
  if (alg1) {
    // H = h: the coarse step is Algorithm 1 on T_h and every correction of Steps 3-4 vanishes
    // identically (the local problems' right-hand sides are the residuals of the converged coarse step in the
    // same space): the composite is the coarse state n+1 (same mesh, same layout)
    for (int f = 0; f < 3; ++f)
      CK(cpya(c->comp2[f], c->cst[sn][f], c->n2p_f * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CK(cpya(c->comp2_u, c->cu[sn], (size_t)D * c->n2c_f * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CK(cpya(c->comp2_p, c->cp[sn], c->n1c_f * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else if (conc) {
    // conduit stage enqueued first (it records evp[2] just before its GMRES launch); the porous stage on st3
    // prepares concurrently and launches its PCG only after that point, on the SMs the GMRES leaves free
    CK(cudaEventRecord(c->evp[0], st));
    c->gate = true;
    conduit_solve_once<D>(c, 1, t, c->cu[sn], c->cp[sn], c->cu[so], c->cst[so][2], c->comp2_u, c->comp2_p);
    CK(cudaStreamWaitEvent(c->st3, c->evp[0], 0));
    {
      StreamSwap sw(c, c->st3);
      porous_stage<D>(c, 1, t, c->cst[sn], c->cst[so], c->cu[so] + (D - 1) * c->n2c_c, c->comp2);
    }
    c->gate = false;
    CK(cudaEventRecord(c->evp[1], c->st3));
    CK(cudaStreamWaitEvent(st, c->evp[1], 0));
  } else {
    porous_stage<D>(c, 1, t, c->cst[sn], c->cst[so], c->cu[so] + (D - 1) * c->n2c_c, c->comp2);
    conduit_solve_once<D>(c, 1, t, c->cu[sn], c->cp[sn], c->cu[so], c->cst[so][2], c->comp2_u, c->comp2_p);
  }
  halo_pack(c);  // a11 (world > 1): the owned values every peer reads, out of the new composite
}

// a11 transfer for the NCCL transport (the local transport's transfer is done by lpfem_step_group), then unpack
void step_exchange(lpfem_ctx* c) {
  if (c->dist.world <= 1) return;
  if (c->dist.transport == LPFEM_TRANSPORT_NCCL) halo_exchange_nccl(c);
  halo_unpack(c);
}

// Step 1 of the next step, overlapped with this fine stage (reads slot n+1, writes n+2).  A non-convergence there
// is not this step's failure: coarse_n stays at n+1 and the next step recomputes (and reports) it.
template <int D>
void step_overlap(lpfem_ctx* c, double dt) {
  CK(cudaEventRecord(c->ev[2], c->st));
  if (c->overlap && !c->kn.no_overlap && !c->alg1k) {
    try {
      coarse_step<D>(c, c->nstep + 1, dt);
    } catch (const Err& e) {
      if (e.code != LPFEM_ENOCONV) throw;
      c->coarse_n = c->nstep + 1;
    }
  }
}

// per-rank convergence of the step's fine solves (host sync)
bool step_verdict(lpfem_ctx* c) {
  const bool alg1 = c->R == 1 && !c->kn.no_alg1_fastpath;
  double maxres[2] = {0, 0};
  bool ok = true;
  if (c->alg1k) {  // the conduit statistics were fetched per Newton iteration
    fetch_stats(c, c->fam[1][0], 0, false, maxres[0], ok);
    ok = ok && c->alg1_ok;
    maxres[1] = c->pending_res[1];
  } else if (!alg1) {
    fetch_stats(c, c->fam[1][0], 0, false, maxres[0], ok);
    fetch_stats(c, c->fam[1][1], 1, false, maxres[1], ok);
  } else {
    CK(cudaStreamSynchronize(c->st));
  }
  c->pending_res[0] = maxres[0];
  c->pending_res[1] = maxres[1];
  c->pending_ok = ok;
  return ok;
}

// NCCL: all ranks commit or none (min over the ranks' verdicts)
bool reduce_verdict_nccl(lpfem_ctx* c, bool ok) {
  if (c->dist.world <= 1 || c->dist.transport != LPFEM_TRANSPORT_NCCL) return ok;
  int h = ok ? 1 : 0;
  CK(cpya(c->dok, &h, sizeof(int), cudaMemcpyHostToDevice, c->st));
  CKN(g_nccl.allReduce(c->dok, c->dok, 1, ncclInt32, ncclMin, c->comm, c->st));
  CK(cpya(&h, c->dok, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return h != 0;
}

void step_end(lpfem_ctx* c, bool ok_all) {
  const bool alg1 = c->R == 1 && !c->kn.no_alg1_fastpath;
  float ms1 = 0, mk0 = 0, mk1 = 0;
  CK(cudaEventElapsedTime(&ms1, c->ev[1], c->ev[2]));
  if (!alg1 && !c->fam[1][0].hs.empty()) CK(cudaEventElapsedTime(&mk0, c->ek[0], c->ek[1]));
  if (!alg1 && !c->fam[1][1].hs.empty()) CK(cudaEventElapsedTime(&mk1, c->ek[2], c->ek[3]));
  if (c->alg1k) mk1 = (float)c->alg1_gm_ms;
  c->stats.t_krylov_ms[0] += mk0;
  c->stats.t_krylov_ms[1] += mk1;
  c->stats.t_fine_ms += ms1;
  c->stats.max_rel_residual[0] = c->pending_res[0];
  c->stats.max_rel_residual[1] = c->pending_res[1];
  if (!ok_all) {
    if (!c->pending_ok) throw Err(LPFEM_ENOCONV, "a Krylov solve did not reach the relative residual (C19); step not committed");
    throw Err(LPFEM_ENOCONV, "a Krylov solve of another rank did not converge (C19); step not committed");
  }
  // commit: the shadow arrays become the state at t_{n+1}
  for (int f = 0; f < 3; ++f) std::swap(c->comp[f], c->comp2[f]);
  std::swap(c->comp_u, c->comp2_u);
  std::swap(c->comp_p, c->comp2_p);
  for (int k = 0; k < 2; ++k) std::swap(c->fam[1][k].ecorr, c->fam[1][k].ecorr2);
  c->t_now = c->pending_t;
  c->nstep++;
  c->stats.steps = c->nstep;
}

template <int D>
void setup(lpfem_ctx* c) {
  upload_tables();
  // reference tensors
  RefT<D>* href = new RefT<D>();
  build_ref<D>(*href);
  c->ref = dalloc<RefT<D>>(1);
  CK(cpy(c->ref, href, sizeof(RefT<D>), cudaMemcpyHostToDevice));
  delete href;
  const lpfem_geometry& g = c->geom;
  const double steps[2] = {c->H, c->h};
  for (int lev = 0; lev < 2; ++lev) {
    const int R = lev == 0 ? 1 : c->R;
    c->Lp[lev].G = make_level(D, g.porous_lo, g.porous_hi, 0, steps[lev], R);
    c->Lc[lev].G = make_level(D, g.conduit_lo, g.conduit_hi, 1, steps[lev], R);
    for (int a = 0; a < 3; ++a) {
      c->Lp[lev].m[a] = c->Lc[lev].m[a] = a < D ? c->m[a] : 1;
      c->Lp[lev].core[a] = c->Lp[lev].G.n[a] / std::max(1, c->Lp[lev].m[a]);
      c->Lc[lev].core[a] = c->Lc[lev].G.n[a] / std::max(1, c->Lc[lev].m[a]);
    }
  }
  for (int a = 0; a < 3; ++a) {
    c->nc_p[a] = c->Lp[0].G.n[a];
    c->nc_c[a] = c->Lc[0].G.n[a];
    c->nf_p[a] = c->Lp[1].G.n[a];
    c->nf_c[a] = c->Lc[1].G.n[a];
  }
  for (int a = 0; a < D; ++a) {
    if (c->nf_p[a] % c->m[a] || c->nf_c[a] % c->m[a])
      throw Err(LPFEM_EMISALIGN, "subdomain grid does not divide the fine mesh");
    if (c->nf_p[a] != c->R * c->nc_p[a] || c->nf_c[a] != c->R * c->nc_c[a])
      throw Err(LPFEM_ENOTDIV, "H/h is not an integer on every axis");
  }
  auto cnt = [&](const int* n, int add, int mul) {
    long long s = 1;
    for (int a = 0; a < D; ++a) s *= (long long)mul * n[a] + add;
    return s;
  };
  c->n2p_f = cnt(c->nf_p, 1, 2);
  c->n2c_f = cnt(c->nf_c, 1, 2);
  c->n1c_f = cnt(c->nf_c, 1, 1);
  c->n2p_c = cnt(c->nc_p, 1, 2);
  c->n2c_c = cnt(c->nc_c, 1, 2);
  c->n1c_c = cnt(c->nc_c, 1, 1);
  c->stats.fine_dofs = 3 * c->n2p_f + D * c->n2c_f + c->n1c_f;
  // coarse families: one system per region
  for (int k = 0; k < 2; ++k) {
    Family& F = c->fam[0][k];
    F.kind = k;
    F.level = 0;
    F.hs.push_back(whole_region(D, k == 0 ? c->Lp[0].G : c->Lc[0].G, k));
    finish_family(D, F);
  }
  // fine families: overlapping subdomains (Algorithm 3 Step 2; C7, C8)
  const int npos = c->m[0] * c->m[1] * (D > 2 ? c->m[2] : 1);
  c->rank_of_pos = placement(region_grid(c, 0), region_grid(c, 1), c->dist.world);  // LPT (halo.h)
  std::vector<int> mine;
  for (int s = 0; s < npos; ++s)
    if (c->rank_of_pos[s] == c->dist.rank) mine.push_back(s);
  for (int k = 0; k < 2; ++k) {
    Family& F = c->fam[1][k];
    F.kind = k;
    F.level = 1;
    const LevelGeom& G = k == 0 ? c->Lp[1].G : c->Lc[1].G;
    for (int s : mine) {
      int pos[3] = {0, 0, 0};
      int rem = s;
      for (int a = 0; a < D; ++a) {
        pos[a] = rem % c->m[a];
        rem /= c->m[a];
      }
      SysDesc S{};
      S.n2 = 1;
      S.n1 = 1;
      std::array<int, 3> cr0 = {0, 0, 0}, cr1 = {0, 0, 0};
      for (int a = 0; a < 3; ++a) {
        S.np[a] = 1;
        if (a >= D) continue;
        const int core = G.n[a] / c->m[a];
        const int c0 = pos[a] * core, c1 = c0 + core;
        const int e0 = std::max(0, c0 - c->ov), e1 = std::min(G.n[a], c1 + c->ov);
        S.c0[a] = e0;
        S.nc[a] = e1 - e0;
        S.np[a] = 2 * S.nc[a] + 1;
        S.art_lo[a] = e0 > 0;
        S.art_hi[a] = e1 < G.n[a];
        S.pos[a] = pos[a];
        S.n2 *= S.np[a];
        S.n1 *= S.nc[a] + 1;
        cr0[a] = c0;
        cr1[a] = c1;
      }
      S.nrows = k == 0 ? S.n2 : D * S.n2 + S.n1;
      S.has_gamma = k == 0 ? (S.c0[D - 1] + S.nc[D - 1] == G.n[D - 1]) : (S.c0[D - 1] == 0);
      S.level = 1;
      F.hs.push_back(S);
      F.sub_region.push_back(k);
      F.sub_pos.push_back(s);
      F.core0.push_back(cr0);
      F.core1.push_back(cr1);
    }
    finish_family(D, F);
  }
  for (int lev = 0; lev < 2; ++lev)
    for (int k = 0; k < 2; ++k) {
      Family& F = c->fam[lev][k];
      if (F.hs.empty()) continue;
      build_pattern<D>(c, F);
      if (k == 1) check_row_len<D>(F);
      alloc_vectors(c, F);
      if (lev == 1) set_order(c, F, false);
      // the fine conduit GMRES multiplies with a node-blocked copy of the operator in 3D (cfg4 GMRES 1597 -> 1290 ms
      // per step); 2D keeps the CSR (cfg2 144 -> 154 ms with it).  LPFEM_NB=0/1 forces either.
      const char* nbk = getenv("LPFEM_NB");
      const bool use_nb = nbk ? atoi(nbk) != 0 : (D == 3 && !getenv("LPFEM_NO_NB"));
      if (lev == 1 && k == 1 && use_nb) build_nb<D>(c, F);
      // 2D: an fp32 copy of the CSR values for the Arnoldi products of the multilevel GMRES (LPFEM_NB_F64=1: none)
      if (lev == 1 && k == 1 && !use_nb && !getenv("LPFEM_NB_F64")) F.aout32 = dalloc<float>(F.nnz);
      // fine porous: fp32 copy of the operators for the PCG's products, with true-residual replacement (experiment
      // LPFEM_PCG_F32=1; measured: +4% / +9% PCG iterations at cfg4 / cfg2 for the same PCG time, so off)
      if (lev == 1 && k == 0 && getenv("LPFEM_PCG_F32")) F.val32 = dalloc<float>(3 * F.nnz);
    }
  // multilevel preconditioner of the fine conduit systems: nested levels r h (r = 2, 4, .. dividing R)
  // and the coarse box at H (mlprec.cuh).  Requires the boxes to lie on coarse grid lines.
  {
    Family& FC = c->fam[1][1];
    bool aligned = !FC.hs.empty();
    for (auto& S : FC.hs)
      for (int a = 0; a < D; ++a) aligned = aligned && S.c0[a] % c->R == 0 && S.nc[a] % c->R == 0;
    std::vector<int> rs;
    for (int r = 2; r < c->R; r *= 2)
      if (c->R % r == 0) rs.push_back(r);
    if (const char* lv = getenv("LPFEM_ML_LEVELS")) {  // experiment: comma-separated intermediate ratios
      rs.clear();
      for (const char* q = lv; *q;) {
        const int r = atoi(q);
        if (r > 1 && r < c->R && c->R % r == 0 && (rs.empty() || r % rs.back() == 0)) rs.push_back(r);
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
    }
    rs.push_back(c->R);
    if (const char* cr = getenv("LPFEM_ML_COARSE")) {  // experiment: coarsest (exactly inverted) level at ratio r < R
      const int r = atoi(cr);
      if (r > 1 && c->R % r == 0) {
        while (!rs.empty() && rs.back() >= r) rs.pop_back();
        rs.push_back(r);
      }
    }
    // R = 1 (H = h): Algorithm 1 on T_h, no fine corrections are solved (do_step), so no multilevel setup
    if (aligned && (int)rs.size() <= NLMAX && c->R > 1) {
      c->nl = (int)rs.size();
      std::vector<long long> poff, aoff;
      long long ptot = 0, atot = 0;
      std::vector<long long> pmax(FC.hs.size(), 0);
      for (int l = 0; l < c->nl; ++l) {
        const int r = rs[l];
        Level& L = c->Llv[l];
        L.G = make_level(D, g.conduit_lo, g.conduit_hi, 1, c->h * r, c->R / r);
        for (int a = 0; a < 3; ++a) {
          L.m[a] = a < D ? c->m[a] : 1;
          L.core[a] = L.G.n[a] / std::max(1, L.m[a]);
        }
        Family& F = c->lvl[l];
        F.kind = 1;
        F.level = 1;
        for (size_t si = 0; si < FC.hs.size(); ++si) {
          SysDesc S = FC.hs[si];
          S.n2 = 1;
          S.n1 = 1;
          for (int a = 0; a < D; ++a) {
            S.c0[a] /= r;
            S.nc[a] /= r;
            S.np[a] = 2 * S.nc[a] + 1;
            S.n2 *= S.np[a];
            S.n1 *= S.nc[a] + 1;
          }
          S.nrows = D * S.n2 + S.n1;
          F.hs.push_back(S);
          long long cells = 1;
          for (int a = 0; a < D; ++a) cells *= S.nc[a];
          pmax[si] = std::max(pmax[si], cells * (D + 1) * p3_of(D));
        }
        finish_family(D, F);
        build_pattern<D>(c, F);
        check_row_len<D>(F);
        alloc_vectors(c, F, true);
        c->ml.q[l] = l == 0 ? r : r / rs[l - 1];
        c->ml.r[l] = r;
        c->ml.direct = getenv("LPFEM_ML_DIRECT") ? atoi(getenv("LPFEM_ML_DIRECT")) : 0;  // 1, 2: see MLArgs
        c->ml.q0[l] = r / rs[0];
        c->ml.st0[l] = nullptr;
        if (c->ml.direct == 2 && l > 0) {
          Stencil* hs0 = new Stencil();
          build_stencil<D>(r / rs[0], *hs0);
          Stencil* ds0 = dalloc<Stencil>(1);
          CK(cpy(ds0, hs0, sizeof(Stencil), cudaMemcpyHostToDevice));
          delete hs0;
          c->stencils.push_back(ds0);
          c->ml.st0[l] = ds0;
        }
        {
          Stencil* hst = new Stencil();
          build_stencil<D>(c->ml.direct == 1 ? r : c->ml.q[l], *hst);
          Stencil* dst = dalloc<Stencil>(1);
          CK(cpy(dst, hst, sizeof(Stencil), cudaMemcpyHostToDevice));
          delete hst;
          c->stencils.push_back(dst);
          c->ml.st[l] = dst;
        }
        c->ml.lsys[l] = F.ds;
        c->ml.LR[l] = F.r;
        c->ml.LZ[l] = F.p;
        c->ml.LS[l] = F.scale;
      }
      for (size_t si = 0; si < FC.hs.size(); ++si) {
        poff.push_back(ptot);
        ptot += pmax[si];
        aoff.push_back(atot);
        const long long n = c->lvl[c->nl - 1].hs[si].nrows;
        atot += n * n;
      }
      aoff.push_back(atot);
      c->haoff = aoff;
      c->part = dalloc<double>(ptot);
      c->aci = dalloc<double>(atot);
      c->abuf = dalloc<double>(atot);
      c->ainv[0] = dalloc<float>(atot);
      c->ainv[1] = dalloc<float>(atot);
      if (getenv("LPFEM_ML_BF16")) {
        c->ainvb[0] = dalloc<__nv_bfloat16>(atot);
        c->ainvb[1] = dalloc<__nv_bfloat16>(atot);
      }
      c->gjperm = dalloc<int>(atot);
      c->dpoff = dalloc<long long>(poff.size());
      c->daoff = dalloc<long long>(aoff.size());
      CK(cpy(c->dpoff, poff.data(), poff.size() * sizeof(long long), cudaMemcpyHostToDevice));
      CK(cpy(c->daoff, aoff.data(), aoff.size() * sizeof(long long), cudaMemcpyHostToDevice));
      int nmax = 1;
      for (auto& S : c->lvl[c->nl - 1].hs) nmax = std::max(nmax, S.nrows);
      c->lpiv = dalloc<int>(nmax + 4096);
      c->linfo = dalloc<int>(1);
      c->ml.nl = c->nl;
      c->ml.aci = c->abuf;  // row-major inverses (k_inv_rowmajor)
      c->ml.aoff = c->daoff;
      c->ml.fsys = FC.ds;
      c->ml.s0 = FC.scale;
      c->ml.nsub = (int)FC.hs.size();
      for (int l = 0; l < NLMAX; ++l) c->ml.lstride[l] = 0;
      c->ml.fstride = 0;
      // ---- porous: same level ratios on the porous boxes (scalar P2, three fields per box)
      Family& FP = c->fam[1][0];
      bool aligned_p = !FP.hs.empty();
      for (auto& S : FP.hs)
        for (int a = 0; a < D; ++a) aligned_p = aligned_p && S.c0[a] % c->R == 0 && S.nc[a] % c->R == 0;
      if (aligned_p && !getenv("LPFEM_NO_POROUS_ML")) {
        c->nlp = c->nl;
        std::vector<long long> aoffp;
        long long atp = 0;
        for (int l = 0; l < c->nlp; ++l) {
          const int r = rs[l];
          Level& L = c->Lplv[l];
          L.G = make_level(D, g.porous_lo, g.porous_hi, 0, c->h * r, c->R / r);
          for (int a = 0; a < 3; ++a) {
            L.m[a] = a < D ? c->m[a] : 1;
            L.core[a] = L.G.n[a] / std::max(1, L.m[a]);
          }
          Family& F = c->plv[l];
          F.kind = 0;
          F.level = 1;
          for (size_t si = 0; si < FP.hs.size(); ++si) {
            SysDesc S = FP.hs[si];
            S.n2 = 1;
            S.n1 = 1;
            for (int a = 0; a < D; ++a) {
              S.c0[a] /= r;
              S.nc[a] /= r;
              S.np[a] = 2 * S.nc[a] + 1;
              S.n2 *= S.np[a];
              S.n1 *= S.nc[a] + 1;
            }
            S.nrows = S.n2;
            F.hs.push_back(S);
          }
          finish_family(D, F);
          build_pattern<D>(c, F);
          alloc_vectors(c, F, true);
          F.dinv = dalloc<double>(3 * F.rows);
          c->mlp.q[l] = c->ml.q[l];
          c->mlp.q0[l] = c->ml.q0[l];
          c->mlp.st0[l] = c->ml.st0[l];
          c->mlp.r[l] = r;
          c->mlp.st[l] = c->ml.st[l];
          c->mlp.lsys[l] = F.ds;
          c->mlp.LR[l] = F.r;
          c->mlp.LZ[l] = F.p;
          c->mlp.LS[l] = F.dinv;
          c->mlp.lstride[l] = F.rows;
        }
        const Family& FL = c->plv[c->nlp - 1];
        for (int f = 0; f < 3; ++f)
          for (size_t si = 0; si < FP.hs.size(); ++si) {
            aoffp.push_back(atp);
            const long long n = FL.hs[si].nrows;
            atp += n * n;
          }
        aoffp.push_back(atp);
        c->haoff_p = aoffp;
        c->aci_p = dalloc<double>(atp);
        c->abuf_p = dalloc<double>(atp);
        c->gjperm_p = dalloc<int>(atp);
        {
          std::vector<SysDesc> h3;
          for (int f = 0; f < 3; ++f)
            for (auto& S3 : FL.hs) h3.push_back(S3);
          c->pds3 = dalloc<SysDesc>(h3.size());
          CK(cpy(c->pds3, h3.data(), h3.size() * sizeof(SysDesc), cudaMemcpyHostToDevice));
        }
        c->daoff_p = dalloc<long long>(aoffp.size());
        CK(cpy(c->daoff_p, aoffp.data(), aoffp.size() * sizeof(long long), cudaMemcpyHostToDevice));
        FP.dinv = dalloc<double>(3 * FP.rows);
        FP.zv = dalloc<double>(3 * FP.rows);
        c->mlp.nl = c->nlp;
        c->mlp.direct = c->ml.direct == 2 ? 2 : 0;
        c->mlp.nsub = (int)FP.hs.size();
        c->mlp.aci = c->abuf_p;  // row-major inverses
        c->mlp.aoff = c->daoff_p;
        c->mlp.fsys = FP.ds;
        c->mlp.s0 = FP.dinv;
        c->mlp.fstride = FP.rows;
      }
    }
  }
  // cluster sizes: spread the systems of a family over the SMs.  Default: from this rank's system counts.
  // world_invariant: from the GLOBAL counts (the world-1 values), identical on every rank and every world size,
  // so that every Krylov reduction has the same order for any world (bitwise world invariance)
  {
    int nsm = 148;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, c->dist.device) == cudaSuccess) nsm = prop.multiProcessorCount;
    c->nsm = nsm;
    const bool inv = c->opts.world_invariant != 0;
    for (int lev = 0; lev < 2; ++lev)
      for (int k = 0; k < 2; ++k) {
        Family& F = c->fam[lev][k];
        const int nsys_loc = std::max<int>(1, (int)F.hk.size());
        const int nsys = (inv && lev == 1) ? (k == 0 ? 3 : 1) * npos : nsys_loc;
        F.nsys_rule = nsys;
        // one 1024-thread CTA per SM: start from nsm / nsys (<= 16, non-portable above 8); the first Krylov
        // launch lowers it until every cluster is resident at once (resident_cluster)
        int cl = std::max(1, std::min(16, nsm / nsys));
        // bandwidth-bound families (largest system > 2M nonzeros: cfg3's 3D boxes) keep the largest power of two
        // and accept a second wave: measured cfg3 (8 systems) cluster 16 in 2 waves 107 ms vs cluster 10 in one
        // wave 145 ms; latency-bound families (cfg1) need one wave: cluster 6 14.6 ms vs 8 in 2 waves 20 ms
        long long nzmax = 0;
        for (long long z : F.sys_nnz) nzmax = std::max(nzmax, z);
        const long long bw_nnz = getenv("LPFEM_BW_NNZ") ? atoll(getenv("LPFEM_BW_NNZ")) : 2000000;  // experiment
        // world_invariant: a rule that does not depend on which boxes this rank holds (3D = bandwidth-bound)
        F.bandwidth_bound = (inv && lev == 1) ? D == 3 : nzmax > bw_nnz;
        if (F.bandwidth_bound) {  // up to two waves: cfg4 cluster 2 / 4 / 8 -> GMRES 1865 / 1777 / 1833 ms
          cl = 1;
          while (cl < 16 && nsys * cl <= nsm) cl *= 2;
        }
        const char* ov = getenv(k == 0 ? "LPFEM_CLUSTER_POROUS" : "LPFEM_CLUSTER_CONDUIT");
        if (ov && lev == 1) cl = std::max(1, std::min(16, atoi(ov)));
        F.cluster = cl;
      }
  }
  // states
  for (int s = 0; s < 3; ++s) {
    for (int f = 0; f < 3; ++f) c->cst[s][f] = dalloc<double>(c->n2p_c);
    c->cu[s] = dalloc<double>(D * c->n2c_c);
    c->cp[s] = dalloc<double>(c->n1c_c);
  }
  c->wpic = dalloc<double>(D * c->n2c_c);
  c->wpic2 = dalloc<double>(D * c->n2c_c);
  c->ppic = dalloc<double>(c->n1c_c);
  c->ppic2 = dalloc<double>(c->n1c_c);
  c->nrm = dalloc<double>(2);
  for (int f = 0; f < 3; ++f) {
    c->comp[f] = dalloc<double>(c->n2p_f);
    c->comp2[f] = dalloc<double>(c->n2p_f);
  }
  c->comp_u = dalloc<double>(D * c->n2c_f);
  c->comp_p = dalloc<double>(c->n1c_f);
  c->comp2_u = dalloc<double>(D * c->n2c_f);
  c->comp2_p = dalloc<double>(c->n1c_f);
  if (c->alg1k) {
    for (int k = 0; k < 2; ++k) {
      c->a1u[k] = dalloc<double>(D * c->n2c_f);
      c->a1p[k] = dalloc<double>(c->n1c_f);
    }
    c->a1uH = dalloc<double>(D * c->n2c_c);
  }
  if (!c->hkmult.empty()) {
    c->kmult = dalloc<double>(c->hkmult.size());
    CK(cpy(c->kmult, c->hkmult.data(), c->hkmult.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  cudaStream_t st = c->st;
  // C12: u_H^0 = I_H u_0, u^h_0 = I_h u_0
  auto init = [&](int lev, double* const* pp, double* u, double* p) {
    const LevelGeom& Gp = c->Lp[lev].G;
    const LevelGeom& Gc = c->Lc[lev].G;
    long long n = lev == 0 ? c->n2p_c : c->n2p_f;
    k_init_p2<D><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Gp, c->pd, c->co, 0, pp[0], pp[1], pp[2], n);
    CKL();
    n = lev == 0 ? c->n2c_c : c->n2c_f;
    k_init_p2<D><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Gc, c->pd, c->co, 1, u, u + n,
                                                               D > 2 ? u + 2 * n : nullptr, n);
    CKL();
    n = lev == 0 ? c->n1c_c : c->n1c_f;
    k_init_p1<D><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Gc, c->pd, c->co, p, n);
    CKL();
  };
  init(0, c->cst[0], c->cu[0], c->cp[0]);
  init(1, c->comp, c->comp_u, c->comp_p);
  {
    const int n = (int)c->fam[0][1].rows;
    if (cusolverDnCreate(&c->sol) != CUSOLVER_STATUS_SUCCESS) throw Err(LPFEM_ECUDA, "cusolverDnCreate");
    cusolverDnSetStream(c->sol, st);
    // the coarse step (one step ahead) runs at the highest stream priority: its small kernels are then dispatched
    // ahead of the fine stage's waiting Krylov clusters instead of queueing behind them (the next fine step waits
    // for it)
    int prio_lo = 0, prio_hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    if (getenv("LPFEM_NO_PRIO")) prio_hi = prio_lo;
    c->prio_hi = prio_hi;
    CK(cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, prio_hi));
    // experiment (LPFEM_PCG_PRIO): the porous stream one priority level above the caller's stream, so that SMs a
    // finished GMRES cluster frees go to waiting PCG CTAs before waiting GMRES clusters (default: equal priority)
    if (getenv("LPFEM_PCG_PRIO") && prio_hi < prio_lo)
      CK(cudaStreamCreateWithPriority(&c->st3, cudaStreamNonBlocking, std::min(prio_lo - 1, std::max(prio_hi + 1, prio_lo - atoi(getenv("LPFEM_PCG_PRIO"))))));
    else
      CK(cudaStreamCreateWithFlags(&c->st3, cudaStreamNonBlocking));
    for (int i = 0; i < 3; ++i) CK(cudaEventCreateWithFlags(&c->evp[i], cudaEventDisableTiming));
    if (const char* gs = getenv("LPFEM_GM_SPLIT")) {
      if (sscanf(gs, "%d:%d:%d", &c->gm_split[0], &c->gm_split[1], &c->gm_split[2]) == 3 && c->gm_split[0] > 0) {
        CK(cudaStreamCreateWithFlags(&c->st4, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&c->evs[i], cudaEventDisableTiming));
      } else {
        c->gm_split[0] = 0;
      }
    }
    {
      auto on = [](const char* k) { return getenv(k) != nullptr; };
      c->kn.verbose = on("LPFEM_VERBOSE");
      // world_invariant: the CTA shared-memory budget (hence the residency check) must not depend on the local boxes
      c->kn.no_smem_pattern = on("LPFEM_NO_SMEM_PATTERN") || c->opts.world_invariant != 0;
      c->kn.cold_start = on("LPFEM_COLD_START");
      c->kn.coarse_full_newton = on("LPFEM_COARSE_FULL_NEWTON");
      c->kn.no_concurrent = on("LPFEM_NO_CONCURRENT");
      c->kn.pcg_ungated = on("LPFEM_PCG_UNGATED");
      c->kn.no_alg1_fastpath = on("LPFEM_NO_ALG1_FASTPATH");
      c->kn.no_overlap = on("LPFEM_NO_OVERLAP");
      if (on("LPFEM_REORTH2")) c->kn.reorth2 = atof(getenv("LPFEM_REORTH2"));
      if (on("LPFEM_GJ_MAX")) c->kn.gj_max = atoi(getenv("LPFEM_GJ_MAX"));
      if (on("LPFEM_PCG_RR")) c->kn.pcg_rr_fac = atof(getenv("LPFEM_PCG_RR"));
    }
    if (getenv("LPFEM_COARSE_PICARD")) c->coarse_newton = 0;
    if (getenv("LPFEM_VEL_W")) c->vw = atof(getenv("LPFEM_VEL_W"));      // experiment knobs
    if (getenv("LPFEM_P_W")) c->pw = atof(getenv("LPFEM_P_W"));
    if (getenv("LPFEM_SCHUR_C")) c->schur_c = atof(getenv("LPFEM_SCHUR_C"));
    if (getenv("LPFEM_WARM_ORDER")) c->warm_order = std::max(1, std::min(2, atoi(getenv("LPFEM_WARM_ORDER"))));
    c->ml_refresh = D == 2 ? 1 : 4;
    if (getenv("LPFEM_ML_REFRESH")) c->ml_refresh = std::max(1, atoi(getenv("LPFEM_ML_REFRESH")));
    for (int i = 0; i < 3; ++i) CK(cudaEventCreateWithFlags(&c->evc[i], cudaEventDefault));
    for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&c->evcp[i], cudaEventDefault));
    if (cusolverDnCreate(&c->sol2) != CUSOLVER_STATUS_SUCCESS) throw Err(LPFEM_ECUDA, "cusolverDnCreate");
    cusolverDnSetStream(c->sol2, c->st2);
    c->dense = dalloc<double>((size_t)n * n);
    c->piv = dalloc<int>(n);
    c->dinfo = dalloc<int>(1);
    if (cusolverDnDgetrf_bufferSize(c->sol, n, n, c->dense, n, &c->lwork) != CUSOLVER_STATUS_SUCCESS)
      throw Err(LPFEM_ECUDA, "cusolverDnDgetrf_bufferSize");
    c->dwork = dalloc<double>(std::max(1, c->lwork));
    if (c->nl > 0) {
      int nmax = 1;
      for (auto& S : c->lvl[c->nl - 1].hs) nmax = std::max(nmax, S.nrows);
      if (c->nlp > 0)
        for (auto& S : c->plv[c->nlp - 1].hs) nmax = std::max(nmax, S.nrows);
      if (cusolverDnDgetrf_bufferSize(c->sol, nmax, nmax, c->abuf, nmax, &c->llwork) != CUSOLVER_STATUS_SUCCESS)
        throw Err(LPFEM_ECUDA, "cusolverDnDgetrf_bufferSize");
      c->lwk = dalloc<double>(std::max(1, c->llwork));
      c->lwk2 = dalloc<double>(std::max(1, c->llwork));
      c->lpiv2 = dalloc<int>(nmax + 4096);
      c->linfo2 = dalloc<int>(1);
      c->nsi = nmax > c->kn.gj_max ? lpfem_ctx::NSI : 0;  // 3D boxes only (2D: batched Gauss-Jordan)
      for (int k = 0; k < c->nsi; ++k) {
        CK(cudaStreamCreateWithPriority(&c->sinv[k], cudaStreamNonBlocking, c->prio_hi));
        if (cusolverDnCreate(&c->hinv[k]) != CUSOLVER_STATUS_SUCCESS) throw Err(LPFEM_ECUDA, "cusolverDnCreate");
        cusolverDnSetStream(c->hinv[k], c->sinv[k]);
        c->lwki[k] = dalloc<double>(std::max(1, c->llwork));
        c->lpivi[k] = dalloc<int>(nmax + 4096);
        c->linfoi[k] = dalloc<int>(1);
      }
      for (int k = 0; k <= c->nsi; ++k) CK(cudaEventCreateWithFlags(&c->einv[k], cudaEventDisableTiming));
    }
  }
  for (int i = 0; i < 4; ++i) {
    CK(cudaEventCreate(&c->ev[i]));
    CK(cudaEventCreate(&c->ek[i]));
  }
  // mode A: e_j^0 = (I_h u_0 - P I_H u_0) on every box node (C12)
  if (c->opts.lag_mode == LPFEM_LAG_SUBDOMAIN) {
    Family& P = c->fam[1][0];
    Family& C = c->fam[1][1];
    if (!P.hs.empty()) {
      PorousPrepArgs A{};
      for (int f = 0; f < 3; ++f) {
        A.coarse_new[f] = c->cst[0][f];
        A.coarse_old[f] = c->cst[0][f];
        A.comp[f] = c->comp[f];
      }
      A.coarse_u_old = c->cu[0];
      for (int a = 0; a < 3; ++a) A.nHu[a] = c->nc_c[a];
      A.Ru = c->R;
      for (int a = 0; a < 3; ++a) {
        A.nHp[a] = c->nc_p[a];
        A.nHc[a] = c->nc_c[a];
        A.np_glob[a] = 2 * c->nf_p[a] + 1;
      }
      A.Rp = c->R;
      A.mode = 0;
      k_porous_prep<D><<<grid_rows(P.maxrows, (int)P.hs.size()), 128, 0, st>>>(
          P.ds, c->Lp[1], c->pd, c->co, A, P.base, P.z, P.lag, P.qf, P.aux, P.rows);
      CKL();
      k_sub<<<(unsigned)((3 * P.rows + 255) / 256), 256, 0, st>>>(P.lag, P.base, P.ecorr, 3 * P.rows);
      CKL();
    }
    if (!C.hs.empty()) {
      ConduitPrepArgs A{};
      A.cu_new = c->cu[0];
      A.cp_new = c->cp[0];
      A.cu_old = c->cu[0];
      A.cpF_old = c->cst[0][2];
      A.comp_u = c->comp_u;
      for (int a = 0; a < 3; ++a) {
        A.nHc[a] = c->nc_c[a];
        A.nHp[a] = c->nc_p[a];
        A.np_glob[a] = 2 * c->nf_c[a] + 1;
      }
      A.R = c->R;
      A.n2_glob = c->n2c_f;
      A.porous_gamma_g = 2 * c->nf_p[D - 1];
      A.mode = 0;
      k_conduit_prep<D><<<grid_rows(C.maxitems, (int)C.hs.size()), 128, 0, st>>>(
          C.ds, c->Lc[1], c->pd, c->co, A, C.base, C.z, C.W, C.lag, C.qf, C.aux);
      CKL();
      k_sub<<<(unsigned)((C.rows + 255) / 256), 256, 0, st>>>(C.lag, C.base, C.ecorr, C.rows);
      CKL();
    }
  }
  if (c->dist.world > 1) setup_multi(c);
  CK(cudaStreamSynchronize(st));
  for (int k = 0; k < 2; ++k) {
    c->stats.n_systems[k] = (long long)c->fam[1][k].hk.size();
    c->stats.n_rows[k] = c->fam[1][k].rows;
    c->stats.nnz[k] = c->fam[1][k].nnz;
  }
}

// buf[f * n + i] = field_f[idx[i]]
__global__ void k_pack(const int* __restrict__ idx, int n, const double* f0, const double* f1, const double* f2,
                       double* __restrict__ buf) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int g = idx[i];
  buf[i] = f0[g];
  if (f1) buf[n + i] = f1[g];
  if (f2) buf[2 * n + i] = f2[g];
}
__global__ void k_unpack(const int* __restrict__ idx, int n, double* f0, double* f1, double* f2,
                         const double* __restrict__ buf) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int g = idx[i];
  f0[g] = buf[i];
  if (f1) f1[g] = buf[n + i];
  if (f2) f2[g] = buf[2 * n + i];
}

int* upload_ints(const std::vector<int>& v) {
  int* d = dalloc<int>(std::max<size_t>(1, v.size()));
  if (!v.empty()) CK(cpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
  return d;
}

RegionGrid region_grid(const lpfem_ctx* c, int reg) {
  RegionGrid G{};
  G.d = c->D;
  for (int a = 0; a < 3; ++a) {
    G.n[a] = a < c->D ? (reg == 0 ? c->nf_p[a] : c->nf_c[a]) : 1;
    G.m[a] = a < c->D ? c->m[a] : 1;
  }
  G.ov = c->ov;
  return G;
}

// ---- local transport: the contexts of one in-process group, by key (dist.nccl_id) and rank
std::mutex g_groups_mu;
std::map<std::string, std::vector<lpfem_ctx*>> g_groups;

std::vector<lpfem_ctx*>& local_group(const lpfem_ctx* c) {
  auto it = g_groups.find(c->group_key);
  if (it == g_groups.end()) throw Err(LPFEM_ESTATE, "local group not registered");
  return it->second;
}

lpfem_ctx* local_peer(const lpfem_ctx* c, int rank) {
  std::vector<lpfem_ctx*>& g = local_group(c);
  if (rank < 0 || rank >= (int)g.size() || !g[rank]) throw Err(LPFEM_ESTATE, "local group incomplete (rank " + std::to_string(rank) + ")");
  return g[rank];
}

const PeerX& peer_entry(const lpfem_ctx* c, int peer) {
  for (const PeerX& X : c->peers)
    if (X.peer == peer) return X;
  throw Err(LPFEM_ESTATE, "no peer entry");
}

void setup_multi(lpfem_ctx* c) {
  const int me = c->dist.rank, W = c->dist.world;
  if (c->dist.transport == LPFEM_TRANSPORT_NCCL) {
    if (!g_nccl.load()) throw Err(LPFEM_ENCCL, "cannot load libnccl.so.2");
    ncclUniqueId id;
    std::memcpy(&id, c->dist.nccl_id, sizeof(id));
    CKN(g_nccl.commInitRank(&c->comm, c->dist.world, id, c->dist.rank));
    c->dok = dalloc<int>(1);
  } else if (c->dist.transport == LPFEM_TRANSPORT_LOCAL) {
    c->group_key.assign((const char*)c->dist.nccl_id, sizeof(c->dist.nccl_id));
    std::lock_guard<std::mutex> lk(g_groups_mu);
    std::vector<lpfem_ctx*>& g = g_groups[c->group_key];
    if (g.empty()) g.assign(W, nullptr);
    if ((int)g.size() != W || g[me]) throw Err(LPFEM_EINVAL, "local group: world or rank clash");
    g[me] = c;
    CK(cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_xdone, cudaEventDisableTiming));
  } else {
    throw Err(LPFEM_EINVAL, "unknown transport");
  }
  plan_region(region_grid(c, 0), c->rank_of_pos, me, W, false, c->plan_p);
  plan_region(region_grid(c, 1), c->rank_of_pos, me, W, false, c->plan_c2);
  plan_region(region_grid(c, 1), c->rank_of_pos, me, W, true, c->plan_c1);
  for (int p = 0; p < W; ++p) {
    if (p == me) continue;
    PeerX X;
    X.peer = p;
    X.np_give = (int)c->plan_p.give[p].size();
    X.nc_give = (int)c->plan_c2.give[p].size();
    X.np_need = (int)c->plan_p.need[p].size();
    X.nc_need = (int)c->plan_c2.need[p].size();
    X.give_p = upload_ints(c->plan_p.give[p]);
    X.give_c = upload_ints(c->plan_c2.give[p]);
    X.need_p = upload_ints(c->plan_p.need[p]);
    X.need_c = upload_ints(c->plan_c2.need[p]);
    X.sbuf = dalloc<double>(3LL * X.np_give + (long long)c->D * X.nc_give + 1);
    X.rbuf = dalloc<double>(3LL * X.np_need + (long long)c->D * X.nc_need + 1);
    c->peers.push_back(X);
  }
  // owned lists of every rank (any rank may be the root of lpfem_get_fields): uploaded once, here
  long long mx = 1;
  for (int p = 0; p < W; ++p) {
    c->own_p.push_back(upload_ints(c->plan_p.owned[p]));
    c->own_c2.push_back(upload_ints(c->plan_c2.owned[p]));
    c->own_c1.push_back(upload_ints(c->plan_c1.owned[p]));
    mx = std::max<long long>(mx, 3LL * c->plan_p.owned[p].size() + (long long)c->D * c->plan_c2.owned[p].size() +
                                     c->plan_c1.owned[p].size());
  }
  c->gbuf_n = mx;
  c->gbuf = dalloc<double>(mx);
}

// a11 after the write-back: the owned values of the lagged fields (3 porous P2 + d velocity P2, C2 mode B) that
// each peer's extended boxes read, out of the new composite (comp2), into one send buffer per peer
void halo_pack(lpfem_ctx* c) {
  if (c->dist.world <= 1) return;
  cudaStream_t st = c->st;
  const int D = c->D;
  const long long n2c = c->n2c_f;
  for (auto& X : c->peers) {
    if (X.np_give) {
      k_pack<<<(X.np_give + 255) / 256, 256, 0, st>>>(X.give_p, X.np_give, c->comp2[0], c->comp2[1], c->comp2[2], X.sbuf);
      CKL();
    }
    if (X.nc_give) {
      k_pack<<<(X.nc_give + 255) / 256, 256, 0, st>>>(X.give_c, X.nc_give, c->comp2_u, c->comp2_u + n2c,
                                                      D > 2 ? c->comp2_u + 2 * n2c : nullptr, X.sbuf + 3LL * X.np_give);
      CKL();
    }
  }
  if (c->dist.transport == LPFEM_TRANSPORT_LOCAL) CK(cudaEventRecord(c->ev_pack, st));
}

// NCCL transport: one group of send/recv per peer pair
void halo_exchange_nccl(lpfem_ctx* c) {
  cudaStream_t st = c->st;
  const int D = c->D;
  CKN(g_nccl.groupStart());
  for (auto& X : c->peers) {
    const size_t ns = 3ULL * X.np_give + (size_t)D * X.nc_give, nr = 3ULL * X.np_need + (size_t)D * X.nc_need;
    if (ns) CKN(g_nccl.send(X.sbuf, ns, ncclFloat64, X.peer, c->comm, st));
    if (nr) CKN(g_nccl.recv(X.rbuf, nr, ncclFloat64, X.peer, c->comm, st));
  }
  CKN(g_nccl.groupEnd());
}

// local transport: copy each peer's send buffer for this rank (packed by the peer's step_begin) into the receive
// buffer, after the peer's pack event
void halo_exchange_local(lpfem_ctx* c) {
  cudaStream_t st = c->st;
  const int D = c->D;
  for (auto& X : c->peers) {
    lpfem_ctx* q = local_peer(c, X.peer);
    const PeerX& Y = peer_entry(q, c->dist.rank);
    const size_t nr = 3ULL * X.np_need + (size_t)D * X.nc_need;
    if (Y.np_give != X.np_need || Y.nc_give != X.nc_need) throw Err(LPFEM_ESTATE, "local halo: list sizes differ");
    CK(cudaStreamWaitEvent(st, q->ev_pack, 0));
    if (nr) CK(cudaMemcpyPeerAsync(X.rbuf, c->dist.device, Y.sbuf, q->dist.device, nr * sizeof(double), st));
  }
  CK(cudaEventRecord(c->ev_xdone, st));
}

void halo_unpack(lpfem_ctx* c) {
  cudaStream_t st = c->st;
  const int D = c->D;
  const long long n2c = c->n2c_f;
  for (auto& X : c->peers) {
    if (X.np_need) {
      k_unpack<<<(X.np_need + 255) / 256, 256, 0, st>>>(X.need_p, X.np_need, c->comp2[0], c->comp2[1], c->comp2[2],
                                                        X.rbuf);
      CKL();
    }
    if (X.nc_need) {
      k_unpack<<<(X.nc_need + 255) / 256, 256, 0, st>>>(X.need_c, X.nc_need, c->comp2_u, c->comp2_u + n2c,
                                                        D > 2 ? c->comp2_u + 2 * n2c : nullptr,
                                                        X.rbuf + 3LL * X.np_need);
      CKL();
    }
  }
}

// pack rank p's owned composite values (committed state) into buf
void pack_owned(lpfem_ctx* q, int p, double* buf, cudaStream_t st) {
  const int D = q->D;
  const long long n2c = q->n2c_f;
  const int np = (int)q->plan_p.owned[p].size(), nc2 = (int)q->plan_c2.owned[p].size(),
            nc1 = (int)q->plan_c1.owned[p].size();
  if (np) k_pack<<<(np + 255) / 256, 256, 0, st>>>(q->own_p[p], np, q->comp[0], q->comp[1], q->comp[2], buf);
  if (nc2)
    k_pack<<<(nc2 + 255) / 256, 256, 0, st>>>(q->own_c2[p], nc2, q->comp_u, q->comp_u + n2c,
                                              D > 2 ? q->comp_u + 2 * n2c : nullptr, buf + 3LL * np);
  if (nc1) k_pack<<<(nc1 + 255) / 256, 256, 0, st>>>(q->own_c1[p], nc1, q->comp_p, nullptr, nullptr,
                                                     buf + 3LL * np + (long long)D * nc2);
  CKL();
}

void unpack_owned(lpfem_ctx* c, int p, const double* buf, cudaStream_t st) {
  const int D = c->D;
  const long long n2c = c->n2c_f;
  const int np = (int)c->plan_p.owned[p].size(), nc2 = (int)c->plan_c2.owned[p].size(),
            nc1 = (int)c->plan_c1.owned[p].size();
  if (np) k_unpack<<<(np + 255) / 256, 256, 0, st>>>(c->own_p[p], np, c->comp[0], c->comp[1], c->comp[2], buf);
  if (nc2)
    k_unpack<<<(nc2 + 255) / 256, 256, 0, st>>>(c->own_c2[p], nc2, c->comp_u, c->comp_u + n2c,
                                                D > 2 ? c->comp_u + 2 * n2c : nullptr, buf + 3LL * np);
  if (nc1) k_unpack<<<(nc1 + 255) / 256, 256, 0, st>>>(c->own_c1[p], nc1, c->comp_p, nullptr, nullptr,
                                                       buf + 3LL * np + (long long)D * nc2);
  CKL();
}

size_t owned_count(const lpfem_ctx* c, int p) {
  return 3ULL * c->plan_p.owned[p].size() + (size_t)c->D * c->plan_c2.owned[p].size() + c->plan_c1.owned[p].size();
}

// gather every rank's owned composite values on root: NCCL send/recv (collective), or (local transport) the root
// packs each peer's values on the peer's stream and copies them over
void gather_root(lpfem_ctx* c, int root) {
  if (c->dist.world <= 1) return;
  cudaStream_t st = c->st;
  const int me = c->dist.rank;
  if (c->dist.transport == LPFEM_TRANSPORT_LOCAL) {
    if (me != root) return;
    for (int p = 0; p < c->dist.world; ++p) {
      if (p == root) continue;
      lpfem_ctx* q = local_peer(c, p);
      CK(cudaSetDevice(q->dist.device));
      pack_owned(q, p, q->gbuf, q->st);
      CK(cudaEventRecord(q->ev_pack, q->st));
      CK(cudaSetDevice(c->dist.device));
      CK(cudaStreamWaitEvent(st, q->ev_pack, 0));
      CK(cudaMemcpyPeerAsync(c->gbuf, c->dist.device, q->gbuf, q->dist.device, owned_count(c, p) * sizeof(double), st));
      unpack_owned(c, p, c->gbuf, st);
      CK(cudaStreamSynchronize(st));  // gbuf is reused for the next peer
    }
    return;
  }
  if (me != root) {
    pack_owned(c, me, c->gbuf, st);
    CKN(g_nccl.send(c->gbuf, owned_count(c, me), ncclFloat64, root, c->comm, st));
    CK(cudaStreamSynchronize(st));
  } else {
    for (int p = 0; p < c->dist.world; ++p) {
      if (p == root) continue;
      CKN(g_nccl.recv(c->gbuf, owned_count(c, p), ncclFloat64, p, c->comm, st));
      unpack_owned(c, p, c->gbuf, st);
    }
    CK(cudaStreamSynchronize(st));
  }
}

// adds this call's kernel launches and host<->device bytes (thread-local counters) to a ctx's statistics
struct Counted {
  lpfem_ctx* c;
  long long l0, h0, d0;
  explicit Counted(lpfem_ctx* cc) : c(cc), l0(tl_launches), h0(tl_h2d), d0(tl_d2h) {}
  ~Counted() {
    if (!c) return;
    c->stats.kernel_launches += tl_launches - l0;
    c->stats.h2d_bytes += tl_h2d - h0;
    c->stats.d2h_bytes += tl_d2h - d0;
  }
};

lpfem_status fail(lpfem_ctx* c, const Err& e) {
  if (c) c->err = e.what();
  return e.code;
}


}  // namespace

// ============================================================================================ C-ABI
extern "C" {

const char* lpfem_status_string(lpfem_status s) {
  switch (s) {
    case LPFEM_OK: return "ok";
    case LPFEM_EINVAL: return "invalid argument";
    case LPFEM_ENOTDIV: return "mesh sizes not integral";
    case LPFEM_EMISALIGN: return "subdomain layout misaligned";
    case LPFEM_ENOCONV: return "solver did not converge";
    case LPFEM_ECUDA: return "CUDA error";
    case LPFEM_ENCCL: return "NCCL error";
    case LPFEM_ENOMEM: return "out of device memory";
    case LPFEM_ESTATE: return "bad state";
  }
  return "unknown";
}

lpfem_status lpfem_nccl_unique_id(unsigned char out[128]) {
  if (!out) return LPFEM_EINVAL;
  if (!g_nccl.load()) return LPFEM_ENCCL;
  return g_nccl.getUniqueId((ncclUniqueId*)out) == ncclSuccess ? LPFEM_OK : LPFEM_ENCCL;
}

lpfem_status lpfem_create(const lpfem_geometry* geom, const lpfem_coeffs* coeffs, const lpfem_data* data, double H,
                          double h, double overlap, const int subdomain_grid[3], const lpfem_opts* opts,
                          const lpfem_dist* dist, lpfem_ctx** out) {
  if (!geom || !coeffs || !data || !subdomain_grid || !opts || !out) return LPFEM_EINVAL;
  *out = nullptr;
  lpfem_ctx* c = new lpfem_ctx();
  try {
    if (geom->dim != 2 && geom->dim != 3) throw Err(LPFEM_EINVAL, "dim must be 2 or 3");
    if (!(H > 0) || !(h > 0) || !(overlap >= 0)) throw Err(LPFEM_EINVAL, "H, h must be > 0 and overlap >= 0");
    c->D = geom->dim;
    c->geom = *geom;
    c->H = H;
    c->h = h;
    c->R = to_int_checked(H / h, LPFEM_ENOTDIV, "H/h");
    to_int_checked(1.0 / h, LPFEM_ENOTDIV, "1/h");
    to_int_checked(1.0 / H, LPFEM_ENOTDIV, "1/H");
    c->ov = (int)std::round(overlap / h);
    if (std::fabs(overlap / h - c->ov) > 1e-9) throw Err(LPFEM_EMISALIGN, "overlap is not a multiple of h");
    for (int a = 0; a < 3; ++a) c->m[a] = a < c->D ? subdomain_grid[a] : 1;
    for (int a = 0; a < c->D; ++a)
      if (c->m[a] < 1) throw Err(LPFEM_EINVAL, "subdomain grid must be >= 1");
    for (int i = 0; i < 3; ++i) {
      c->co.phiC[i] = coeffs->phi[i] * coeffs->C[i];
      c->co.k[i] = coeffs->k[i];
    }
    c->co.sigma = coeffs->sigma;
    c->co.sigma_star = coeffs->sigma_star;
    c->co.mu = coeffs->mu_tilde;
    c->co.nu = coeffs->nu;
    c->co.rho = coeffs->rho;
    c->co.alpha = coeffs->alpha;
    c->co.eta = coeffs->eta;
    c->pd.kind = data->problem;
    c->pd.peak = data->inflow_peak;
    c->pd.cval = data->const_value;
    if (c->pd.kind < 0 || c->pd.kind > 3) throw Err(LPFEM_EINVAL, "unknown problem");
    c->opts = *opts;
    if (c->opts.krylov_rtol <= 0) c->opts.krylov_rtol = 1e-12;
    if (c->opts.max_iter <= 0) c->opts.max_iter = 20000;
    if (c->opts.picard_rtol <= 0) c->opts.picard_rtol = 1e-13;
    if (c->opts.picard_max <= 0) c->opts.picard_max = 50;
    if (c->opts.gmres_restart != 0 && c->opts.gmres_restart != GM)
      throw Err(LPFEM_EINVAL, "gmres_restart: 0 (default) or the compiled restart length " + std::to_string(GM) +
                                  " (LPFEM_GM at build time)");
    c->opts.gmres_restart = GM;
    if (c->opts.algorithm == 0) c->opts.algorithm = 3;
    if (c->opts.algorithm != 1 && c->opts.algorithm != 3) throw Err(LPFEM_EINVAL, "algorithm: 1 or 3");
    if (c->opts.algorithm == 1 && c->R > 1) {  // Algorithm 1 at scale: whole-region systems, H = preconditioner level
      for (int a = 0; a < c->D; ++a)
        if (c->m[a] != 1) throw Err(LPFEM_EINVAL, "algorithm 1: subdomain grid must be 1 (whole regions)");
      if (c->ov != 0) throw Err(LPFEM_EINVAL, "algorithm 1: overlap must be 0");
      c->alg1k = true;
    }
    if (dist) {
      c->dist = *dist;
    } else {
      c->dist.rank = 0;
      c->dist.world = 1;
      c->dist.device = 0;
      c->dist.transport = LPFEM_TRANSPORT_NCCL;
    }
    if (c->dist.world == 1) c->group_key.clear();
    if (c->dist.world < 1 || c->dist.rank < 0 || c->dist.rank >= c->dist.world) throw Err(LPFEM_EINVAL, "bad dist");
    CK(cudaSetDevice(c->dist.device));
    c->st = (cudaStream_t)c->dist.cuda_stream;
    if (coeffs->k_mult) {
      long long ncells = 1;
      for (int a = 0; a < c->D; ++a)
        ncells *= to_int_checked((geom->porous_hi[a] - geom->porous_lo[a]) / H, LPFEM_ENOTDIV, "porous extent / H");
      c->hkmult.assign(coeffs->k_mult, coeffs->k_mult + ncells);
    }
    {
      Counted cnt(c);
      if (c->D == 2) setup<2>(c); else setup<3>(c);
    }
    *out = c;
    return LPFEM_OK;
  } catch (const Err& e) {
    lpfem_status s = e.code;
    fprintf(stderr, "lpfem_create: %s\n", e.what());
    lpfem_destroy(c);
    return s;
  }
}

lpfem_status lpfem_step(lpfem_ctx* c, double dt) {
  if (!c) return LPFEM_EINVAL;
  if (!(dt > 0)) {
    c->err = "dt must be > 0";
    return LPFEM_EINVAL;
  }
  if (c->dist.world > 1 && c->dist.transport == LPFEM_TRANSPORT_LOCAL) {
    c->err = "local-transport contexts are stepped by lpfem_step_group";
    return LPFEM_ESTATE;
  }
  Counted cnt(c);
  try {
    if (c->D == 2) step_begin<2>(c, dt); else step_begin<3>(c, dt);
    step_exchange(c);
    if (c->D == 2) step_overlap<2>(c, dt); else step_overlap<3>(c, dt);
    const bool ok = reduce_verdict_nccl(c, step_verdict(c));
    step_end(c, ok);
    return LPFEM_OK;
  } catch (const Err& e) {
    return fail(c, e);
  }
}

lpfem_status lpfem_step_group(lpfem_ctx* const* ctxs, int n, double dt) {
  if (!ctxs || n < 1 || !(dt > 0)) return LPFEM_EINVAL;
  // the contexts must be exactly the ranks of one local group
  std::vector<lpfem_ctx*> g(n, nullptr);
  for (int i = 0; i < n; ++i) {
    lpfem_ctx* c = ctxs[i];
    if (!c || c->dist.world != n || c->dist.rank < 0 || c->dist.rank >= n || g[c->dist.rank]) return LPFEM_EINVAL;
    if (n > 1 && c->dist.transport != LPFEM_TRANSPORT_LOCAL) return LPFEM_EINVAL;
    if (c->group_key != ctxs[0]->group_key) return LPFEM_EINVAL;
    g[c->dist.rank] = c;
  }
  lpfem_ctx* cur = g[0];
  Counted cnt(g[0]);  // the group's launches and copies are accounted on rank 0
  try {
    for (lpfem_ctx* c : g) {  // phase 1: coarse (if needed), fine stage, write-back, pack
      cur = c;
      if (c->D == 2) step_begin<2>(c, dt); else step_begin<3>(c, dt);
    }
    if (n > 1) {
      for (lpfem_ctx* c : g) {  // phase 2: transfers (after every peer's pack) and unpack
        cur = c;
        CK(cudaSetDevice(c->dist.device));
        halo_exchange_local(c);
        halo_unpack(c);
      }
      // a peer's send buffers are rewritten by its next pack only after every copy out of them is done
      for (lpfem_ctx* c : g) {
        cur = c;
        CK(cudaSetDevice(c->dist.device));
        for (lpfem_ctx* q : g)
          if (q != c) CK(cudaStreamWaitEvent(c->st, q->ev_xdone, 0));
      }
    }
    bool ok = true;
    for (lpfem_ctx* c : g) {  // phase 3: coarse step ahead, verdicts
      cur = c;
      if (c->D == 2) step_overlap<2>(c, dt); else step_overlap<3>(c, dt);
    }
    for (lpfem_ctx* c : g) {
      cur = c;
      ok = step_verdict(c) && ok;
    }
    lpfem_status st = LPFEM_OK;
    for (lpfem_ctx* c : g) {  // phase 4: all commit or none
      try {
        step_end(c, ok);
      } catch (const Err& e) {
        st = fail(c, e);
      }
    }
    return st;
  } catch (const Err& e) {
    for (lpfem_ctx* c : g) c->err = e.what();
    return fail(cur, e);
  }
}

lpfem_status lpfem_inject_fault(lpfem_ctx* c, int family, int max_iter) {
  if (!c || family < 0 || family > 1) return LPFEM_EINVAL;
  c->fault_maxit[family] = max_iter > 0 ? max_iter : 0;
  return LPFEM_OK;
}

lpfem_status lpfem_get_sizes(const lpfem_ctx* c, long long n_nodes_p2[2], long long n_nodes_p1[2]) {
  if (!c || !n_nodes_p2 || !n_nodes_p1) return LPFEM_EINVAL;
  n_nodes_p2[0] = c->n2p_f;
  n_nodes_p2[1] = c->n2c_f;
  n_nodes_p1[0] = 0;
  n_nodes_p1[1] = c->n1c_f;
  return LPFEM_OK;
}

static lpfem_status copy_out(lpfem_ctx* c, double* dst, const double* src, long long n, int on_device) {
  if (!dst) return LPFEM_OK;
  cudaError_t e = cpya(dst, src, n * sizeof(double), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st);
  if (e != cudaSuccess) {
    c->err = cudaGetErrorString(e);
    return LPFEM_ECUDA;
  }
  return LPFEM_OK;
}

lpfem_status lpfem_get_fields(lpfem_ctx* c, double* pF, double* pf, double* pm, double* u, double* p, int on_device,
                              int root) {
  if (!c) return LPFEM_EINVAL;
  if (root < 0 || root >= c->dist.world) return LPFEM_EINVAL;
  Counted cnt(c);
  try {
    CK(cudaSetDevice(c->dist.device));
    gather_root(c, root);
  } catch (const Err& e) {
    return fail(c, e);
  }
  if (c->dist.rank != root) return LPFEM_OK;
  lpfem_status s;
  if ((s = copy_out(c, pF, c->comp[2], c->n2p_f, on_device))) return s;
  if ((s = copy_out(c, pf, c->comp[1], c->n2p_f, on_device))) return s;
  if ((s = copy_out(c, pm, c->comp[0], c->n2p_f, on_device))) return s;
  if ((s = copy_out(c, u, c->comp_u, c->D * c->n2c_f, on_device))) return s;
  if ((s = copy_out(c, p, c->comp_p, c->n1c_f, on_device))) return s;
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return LPFEM_ECUDA;
  return LPFEM_OK;
}

lpfem_status lpfem_get_coarse_fields(lpfem_ctx* c, double* pF, double* pf, double* pm, double* u, double* p) {
  if (!c) return LPFEM_EINVAL;
  lpfem_status s;
  const int k = (int)(c->nstep % 3);
  if (cudaStreamSynchronize(c->st2) != cudaSuccess) return LPFEM_ECUDA;
  if ((s = copy_out(c, pF, c->cst[k][2], c->n2p_c, 0))) return s;
  if ((s = copy_out(c, pf, c->cst[k][1], c->n2p_c, 0))) return s;
  if ((s = copy_out(c, pm, c->cst[k][0], c->n2p_c, 0))) return s;
  if ((s = copy_out(c, u, c->cu[k], c->D * c->n2c_c, 0))) return s;
  if ((s = copy_out(c, p, c->cp[k], c->n1c_c, 0))) return s;
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return LPFEM_ECUDA;
  return LPFEM_OK;
}

lpfem_status lpfem_get_mesh(const lpfem_ctx* c, int which, double* coords, int* cells, long long n_out[2]) {
  if (!c || !n_out || which < 0 || which > 3) return LPFEM_EINVAL;
  const int D = c->D;
  const int lev = which / 2, reg = which % 2;
  const LevelGeom& G = reg == 0 ? c->Lp[lev].G : c->Lc[lev].G;
  int np[3] = {1, 1, 1};
  long long n2 = 1, ncell = 1;
  for (int a = 0; a < D; ++a) {
    np[a] = 2 * G.n[a] + 1;
    n2 *= np[a];
    ncell *= G.n[a];
  }
  KuhnTables T;
  build_kuhn(D, T);
  const int nt = nt_of(D), N = n2_of(D);
  n_out[0] = n2;
  n_out[1] = ncell * nt;
  if (coords) {
    for (long long i = 0; i < n2; ++i) {
      int g[3] = {0, 0, 0};
      unlex<3>(i, np, g);
      for (int a = 0; a < D; ++a) {
        volatile double prod = (double)g[a] * G.hg[a];  // no contraction: lo + g * step (C21)
        coords[i * D + a] = G.lo[a] + prod;
      }
    }
  }
  if (cells) {
    for (long long k = 0; k < ncell; ++k) {
      int cc[3] = {0, 0, 0};
      int nn[3] = {G.n[0], G.n[1], G.n[2]};
      unlex<3>(k, nn, cc);
      for (int t = 0; t < nt; ++t)
        for (int j = 0; j < N; ++j) {
          int v[3] = {0, 0, 0};
          for (int a = 0; a < D; ++a) v[a] = 2 * cc[a] + T.off[t][j][a];
          long long idx = 0, s = 1;
          for (int a = 0; a < D; ++a) {
            idx += v[a] * s;
            s *= np[a];
          }
          cells[(k * nt + t) * N + j] = (int)idx;
        }
    }
  }
  return LPFEM_OK;
}

lpfem_status lpfem_get_layout(const lpfem_ctx* c, int* region, int* pos, int* core0, int* core1, int* box0, int* box1,
                              int* n_out) {
  if (!c || !n_out) return LPFEM_EINVAL;
  int n = 0;
  for (int k = 0; k < 2; ++k) {
    const Family& F = c->fam[1][k];
    for (size_t s = 0; s < F.hs.size(); ++s, ++n) {
      if (region) region[n] = k;
      if (pos) pos[n] = F.sub_pos[s];
      for (int a = 0; a < 3; ++a) {
        if (core0) core0[3 * n + a] = F.core0[s][a];
        if (core1) core1[3 * n + a] = F.core1[s][a];
        if (box0) box0[3 * n + a] = F.hs[s].c0[a];
        if (box1) box1[3 * n + a] = F.hs[s].c0[a] + F.hs[s].nc[a];
      }
    }
  }
  *n_out = n;
  return LPFEM_OK;
}

lpfem_status lpfem_get_stats(const lpfem_ctx* c, lpfem_stats* out) {
  if (!c || !out) return LPFEM_EINVAL;
  *out = c->stats;
  return LPFEM_OK;
}

lpfem_status lpfem_get_system(lpfem_ctx* c, int family, int local_index, int field, long long* nrows, long long* nnz,
                              long long* rowptr, int* col, double* val, double* rhs, double* x) {
  if (!c || family < 0 || family > 1 || !nrows || !nnz) return LPFEM_EINVAL;
  Family& F = c->fam[1][family];
  if (local_index < 0 || local_index >= (int)F.hs.size()) return LPFEM_EINVAL;
  if (family == 0 && (field < 0 || field > 2)) return LPFEM_EINVAL;
  const SysDesc& S = F.hs[local_index];
  std::vector<long long> rp(S.nrows + 1);
  if (cpy(rp.data(), F.rowptr + S.row_off, (S.nrows + 1) * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return LPFEM_ECUDA;
  *nrows = S.nrows;
  *nnz = rp[S.nrows] - rp[0];
  if (rowptr)
    for (int i = 0; i <= S.nrows; ++i) rowptr[i] = rp[i] - rp[0];
  const long long voff = family == 0 ? field * F.nnz : 0;
  const long long roff = (family == 0 ? field * F.rows : 0) + S.row_off;
  const double* vsrc = family == 0 ? F.val : F.aout;
  if (col && cpy(col, F.col + rp[0], *nnz * sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return LPFEM_ECUDA;
  if (val && cpy(val, vsrc + voff + rp[0], *nnz * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return LPFEM_ECUDA;
  if (rhs && cpy(rhs, F.rhs + roff, S.nrows * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return LPFEM_ECUDA;
  if (x && cpy(x, F.x + roff, S.nrows * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) return LPFEM_ECUDA;
  return LPFEM_OK;
}

lpfem_status lpfem_bench_spmv(lpfem_ctx* c, int family, int reps, int flush, double* ms_per_rep,
                              double* bytes_per_rep) {
  if (!c || family < 0 || family > 1 || reps < 1 || !ms_per_rep || !bytes_per_rep) return LPFEM_EINVAL;
  try {
    CK(cudaSetDevice(c->dist.device));
    Family& F = c->fam[1][family];
    if (F.hk.empty() || F.nnz == 0) throw Err(LPFEM_ESTATE, "family has no systems on this rank");
    const double* val = family == 0 ? F.val : F.aout;
    const double* x = F.rhs;
    double* y = family == 0 ? F.q : F.W;
    constexpr int NT = 512;
    int tpr = family == 0 ? (c->D == 2 ? 4 : 8) : (c->D == 2 ? TPR2 : TPR3);
    if (family == 1 && F.nbval) {  // the node-blocked operator the GMRES multiplies with
      // the values the GMRES's Arnoldi products read: the fp32 copy when there is one
      const NBMat B{F.nbval, F.nbval32, F.nbcol, F.nbvptr, F.nbcptr, F.nblen, F.nbcol16, F.nbcbase};
      int maxi = 0;
      double bytes = 0.0;
      for (size_t i = 0; i < F.hk.size(); ++i) {
        const KSys& K = F.hk[i];
        maxi = std::max(maxi, K.n2 + K.n1);
      }
      bytes = (F.nbval32 ? 4.0 : 8.0) * F.nnz + (F.nbcol16 ? 2.0 * F.nb_ncols + 8.0 * F.nb_items : 4.0 * F.nb_ncols) +
              24.0 * F.nb_items + 16.0 * F.rows;
      const int ipc = 4 * NT / tpr;
      const dim3 grid((maxi + ipc - 1) / ipc, (unsigned)F.hk.size());
      void* fb = nullptr;
      const size_t fbytes = 512u << 20;
      if (flush) CK(cudaMalloc(&fb, fbytes));
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      double tot = 0.0;
      for (int r = 0; r < reps; ++r) {
        if (flush) CK(cudaMemsetAsync(fb, r & 0xff, fbytes, c->st));
        CK(cudaEventRecord(e0, c->st));
        if (c->D == 2 && F.nbval32)
          k_spmv_nb_family<NT, TPR2, 2, float><<<grid, NT, 0, c->st>>>(F.dk, B, F.nbval32, F.rhs, F.W, ipc);
        else if (c->D == 2)
          k_spmv_nb_family<NT, TPR2, 2, double><<<grid, NT, 0, c->st>>>(F.dk, B, F.nbval, F.rhs, F.W, ipc);
        else if (F.nbval32)
          k_spmv_nb_family<NT, TPR3, 3, float><<<grid, NT, 0, c->st>>>(F.dk, B, F.nbval32, F.rhs, F.W, ipc);
        else
          k_spmv_nb_family<NT, TPR3, 3, double><<<grid, NT, 0, c->st>>>(F.dk, B, F.nbval, F.rhs, F.W, ipc);
        CKL();
        CK(cudaEventRecord(e1, c->st));
        CK(cudaEventSynchronize(e1));
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        tot += ms;
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      if (fb) cudaFree(fb);
      *ms_per_rep = tot / reps;
      *bytes_per_rep = bytes;
      return LPFEM_OK;
    }
    if (getenv("LPFEM_SPMV_TPR")) tpr = atoi(getenv("LPFEM_SPMV_TPR"));  // experiment
    const int rpc = 4 * NT / tpr;
    int maxr = 0;
    double bytes = 0.0;
    for (size_t i = 0; i < F.hk.size(); ++i) {
      const KSys& K = F.hk[i];
      maxr = std::max(maxr, K.nrows);
      const double nz = (double)(F.hrp[K.prow_off + K.nrows] - F.hrp[K.prow_off]);
      bytes += (family == 1 && F.aout32 ? 8.0 : 12.0) * nz + 8.0 * (K.nrows + 1) + 16.0 * K.nrows;
    }
    const dim3 grid((maxr + rpc - 1) / rpc, (unsigned)F.hk.size());
    void* fb = nullptr;
    const size_t fbytes = 512u << 20;
    if (flush) CK(cudaMalloc(&fb, fbytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double tot = 0.0;
    for (int r = 0; r < reps; ++r) {
      if (flush) CK(cudaMemsetAsync(fb, r & 0xff, fbytes, c->st));
      CK(cudaEventRecord(e0, c->st));
      // the Krylov kernels' choice: pipelined rows (U = 4) for the porous family and the 2D conduit, plain 3D conduit
      const int pu = getenv("LPFEM_SPMV_PIPE") ? atoi(getenv("LPFEM_SPMV_PIPE")) : (family == 0 || c->D == 2 ? 4 : 0);
      // (the 2D conduit: the fp32 values the GMRES's Arnoldi products read)
#define LP_SPMV(T, P)                                                                                            \
  ((family == 1 && F.aout32)                                                                                     \
       ? k_spmv_family<NT, T, P, float><<<grid, NT, 0, c->st>>>(F.dk, F.rowptr, F.col, F.aout32, x, y, rpc)     \
       : k_spmv_family<NT, T, P><<<grid, NT, 0, c->st>>>(F.dk, F.rowptr, F.col, val, x, y, rpc))
      if (pu == 4) {
        if (tpr == 4) LP_SPMV(4, 4);
        else if (tpr == 8) LP_SPMV(8, 4);
        else if (tpr == 16) LP_SPMV(16, 4);
        else LP_SPMV(32, 4);
      } else if (pu == 8) {
        if (tpr == 4) LP_SPMV(4, 8);
        else if (tpr == 8) LP_SPMV(8, 8);
        else if (tpr == 16) LP_SPMV(16, 8);
        else LP_SPMV(32, 8);
      } else {
        if (tpr == 4) LP_SPMV(4, 0);
        else if (tpr == 8) LP_SPMV(8, 0);
        else LP_SPMV(16, 0);
      }
#undef LP_SPMV
      CKL();
      CK(cudaEventRecord(e1, c->st));
      CK(cudaEventSynchronize(e1));
      float ms = 0.0f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      tot += ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (fb) cudaFree(fb);
    *ms_per_rep = tot / reps;
    *bytes_per_rep = bytes;
    return LPFEM_OK;
  } catch (const Err& e) {
    return fail(c, e);
  }
}

static bool plan_grids(int dim, const int* ncp, const int* ncc, const int* grid, int ov, RegionGrid& Gp, RegionGrid& Gc) {
  if (!ncp || !ncc || !grid || dim < 2 || dim > 3 || ov < 0) return false;
  for (RegionGrid* G : {&Gp, &Gc}) {
    const int* n = G == &Gp ? ncp : ncc;
    G->d = dim;
    G->ov = ov;
    for (int a = 0; a < 3; ++a) {
      G->n[a] = a < dim ? n[a] : 1;
      G->m[a] = a < dim ? grid[a] : 1;
      if (a < dim && (G->m[a] < 1 || G->n[a] < 1 || G->n[a] % G->m[a])) return false;
    }
  }
  return true;
}

lpfem_status lpfem_placement(int dim, const int n_cells_p[3], const int n_cells_c[3], const int subdomain_grid[3],
                             int overlap_cells, int world, int* rank_of_pos) {
  RegionGrid Gp{}, Gc{};
  if (world < 1 || !rank_of_pos || !plan_grids(dim, n_cells_p, n_cells_c, subdomain_grid, overlap_cells, Gp, Gc))
    return LPFEM_EINVAL;
  const std::vector<int> r = placement(Gp, Gc, world);
  std::copy(r.begin(), r.end(), rank_of_pos);
  return LPFEM_OK;
}

lpfem_status lpfem_halo_plan(int dim, const int n_cells_p[3], const int n_cells_c[3], const int subdomain_grid[3],
                             int overlap_cells, int region, int rank, int world, int vertex_only, int kind, int peer,
                             int* out, long long* n_out) {
  RegionGrid Gp{}, Gc{};
  if (!n_out || world < 1 || rank < 0 || rank >= world || peer < 0 || peer >= world || kind < 0 || kind > 2 ||
      region < 0 || region > 1 || !plan_grids(dim, n_cells_p, n_cells_c, subdomain_grid, overlap_cells, Gp, Gc))
    return LPFEM_EINVAL;
  HaloPlan P;
  plan_region(region == 0 ? Gp : Gc, placement(Gp, Gc, world), rank, world, vertex_only != 0, P);
  const std::vector<int>& v = kind == 0 ? P.need[peer] : (kind == 1 ? P.give[peer] : P.owned[peer]);
  *n_out = (long long)v.size();
  if (out) std::copy(v.begin(), v.end(), out);
  return LPFEM_OK;
}

const char* lpfem_last_error(const lpfem_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

void lpfem_destroy(lpfem_ctx* c) {
  if (!c) return;
  for (int lev = 0; lev < 2; ++lev)
    for (int k = 0; k < 2; ++k) c->fam[lev][k].free_all();
  for (int s = 0; s < 3; ++s) {
    for (int f = 0; f < 3; ++f)
      if (c->cst[s][f]) cudaFree(c->cst[s][f]);
    if (c->cu[s]) cudaFree(c->cu[s]);
    if (c->cp[s]) cudaFree(c->cp[s]);
  }
  for (int l = 0; l < NLMAX; ++l) c->lvl[l].free_all();
  for (int l = 0; l < NLMAX; ++l) c->plv[l].free_all();
  {
    void* pp[] = {c->aci_p, c->abuf_p, c->daoff_p};
    for (void* p : pp)
      if (p) cudaFree(p);
  }
  for (void* p : c->stencils) cudaFree(p);
  for (auto& X : c->peers) {
    void* xp[] = {X.give_p, X.give_c, X.need_p, X.need_c, X.sbuf, X.rbuf};
    for (void* p : xp)
      if (p) cudaFree(p);
  }
  for (auto* v : {&c->own_p, &c->own_c2, &c->own_c1})
    for (int* p : *v)
      if (p) cudaFree(p);
  if (c->gbuf) cudaFree(c->gbuf);
  if (c->dok) cudaFree(c->dok);
  if (!c->group_key.empty()) {  // leave the local group
    std::lock_guard<std::mutex> lk(g_groups_mu);
    auto it = g_groups.find(c->group_key);
    if (it != g_groups.end()) {
      for (auto& q : it->second)
        if (q == c) q = nullptr;
      bool empty = true;
      for (auto* q : it->second) empty = empty && !q;
      if (empty) g_groups.erase(it);
    }
  }
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_xdone) cudaEventDestroy(c->ev_xdone);
  if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  if (c->st2) cudaStreamSynchronize(c->st2);
  if (c->st3) cudaStreamSynchronize(c->st3);
  {
    void* mp[] = {c->gjperm, c->gjperm_p, c->pds3, c->part, c->aci, c->abuf, c->lwk, c->dpoff, c->daoff, c->lpiv, c->linfo,
                  c->ainv[0], c->ainv[1], c->ainvb[0], c->ainvb[1], c->cstab, c->lwk2, c->lpiv2, c->linfo2};
    for (void* p : mp)
      if (p) cudaFree(p);
  }
  if (c->sol) cusolverDnDestroy(c->sol);
  if (c->sol2) cusolverDnDestroy(c->sol2);
  for (int k = 0; k < lpfem_ctx::NSI; ++k) {
    if (c->sinv[k]) cudaStreamSynchronize(c->sinv[k]);
    if (c->hinv[k]) cusolverDnDestroy(c->hinv[k]);
    if (c->sinv[k]) cudaStreamDestroy(c->sinv[k]);
    void* q[] = {c->lwki[k], c->lpivi[k], c->linfoi[k]};
    for (void* p : q)
      if (p) cudaFree(p);
  }
  for (int k = 0; k <= lpfem_ctx::NSI; ++k)
    if (c->einv[k]) cudaEventDestroy(c->einv[k]);
  if (c->st2) {
    cudaStreamSynchronize(c->st2);
    cudaStreamDestroy(c->st2);
  }
  if (c->st3) cudaStreamDestroy(c->st3);
  if (c->st4) cudaStreamDestroy(c->st4);
  for (auto e : c->evs)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 3; ++i)
    if (c->evp[i]) cudaEventDestroy(c->evp[i]);
  for (int i = 0; i < 3; ++i)
    if (c->evc[i]) cudaEventDestroy(c->evc[i]);
  for (int i = 0; i < 2; ++i)
    if (c->evcp[i]) cudaEventDestroy(c->evcp[i]);
  void* ptrs[] = {c->dense, c->dwork, c->piv, c->dinfo, c->wpic, c->wpic2, c->ppic, c->ppic2, c->nrm, c->comp[0], c->comp[1], c->comp[2], c->comp_u,
                  c->comp_p, c->comp2[0], c->comp2[1], c->comp2[2], c->comp2_u, c->comp2_p, c->kmult, c->ref,
                  c->a1u[0], c->a1u[1], c->a1p[0], c->a1p[1], c->a1uH};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (int i = 0; i < 4; ++i) {
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    if (c->ek[i]) cudaEventDestroy(c->ek[i]);
  }
  delete c;
}

}  // extern "C"
