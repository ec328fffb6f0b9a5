"""paper_2311_05170_b200 -- B200-native local parallel two-grid FEM (arXiv 2311.05170, Algorithm 3).

Thin ctypes binding over the C-ABI declared in ``include/lpfem.h`` (argument marshalling only:
every step of the path runs in the CUDA kernels of ``liblpfem.so``).  There is no CPU fallback:
importing works without a GPU, but creating a context fails loudly when the library or a CUDA
device is missing.

    from paper_2311_05170_b200 import LPFEM
    import lpfem_inputs
    sim = LPFEM(lpfem_inputs.config(1))
    for _ in range(10):
        sim.step()
    f = sim.fields()          # dict of numpy arrays: pF, pf, pm, u (d, n), p
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LPFEM_LIB") or os.path.join(HERE, "liblpfem.so")  # override: experiment builds

PROB = {"mms": 0, "injection": 1, "constant": 2, "mms_steady": 3}
LAG = {"composite": 0, "subdomain": 1}
STATUS = ["ok", "einval", "enotdiv", "emisalign", "enoconv", "ecuda", "enccl", "enomem", "estate"]

# Exported symbols (kept in sync with include/lpfem.h; checked by tests/test_abi.py)
SYMBOLS = ["lpfem_nccl_unique_id", "lpfem_create", "lpfem_step", "lpfem_step_group", "lpfem_inject_fault",
           "lpfem_get_sizes", "lpfem_get_fields", "lpfem_get_coarse_fields", "lpfem_get_mesh", "lpfem_get_layout",
           "lpfem_get_stats", "lpfem_get_system", "lpfem_placement", "lpfem_halo_plan", "lpfem_last_error",
           "lpfem_status_string", "lpfem_destroy", "lpfem_bench_spmv"]
TRANSPORT = {"nccl": 0, "local": 1}


class Geometry(C.Structure):
    _fields_ = [("dim", C.c_int), ("porous_lo", C.c_double * 3), ("porous_hi", C.c_double * 3),
                ("conduit_lo", C.c_double * 3), ("conduit_hi", C.c_double * 3)]


class Coeffs(C.Structure):
    _fields_ = [("phi", C.c_double * 3), ("C", C.c_double * 3), ("k", C.c_double * 3), ("sigma", C.c_double),
                ("sigma_star", C.c_double), ("mu_tilde", C.c_double), ("nu", C.c_double), ("rho", C.c_double),
                ("alpha", C.c_double), ("eta", C.c_double), ("k_mult", C.POINTER(C.c_double))]


class Data(C.Structure):
    _fields_ = [("problem", C.c_int), ("inflow_peak", C.c_double), ("const_value", C.c_double)]


class Opts(C.Structure):
    _fields_ = [("lag_mode", C.c_int), ("krylov_rtol", C.c_double), ("max_iter", C.c_int), ("gmres_restart", C.c_int),
                ("picard_rtol", C.c_double), ("picard_max", C.c_int), ("world_invariant", C.c_int),
                ("algorithm", C.c_int)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("device", C.c_int), ("nccl_id", C.c_ubyte * 128),
                ("cuda_stream", C.c_void_p), ("transport", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("steps", C.c_longlong), ("fine_iters", C.c_longlong * 2), ("fine_max_iters", C.c_longlong * 2),
                ("coarse_iters", C.c_longlong * 2), ("picard_iters", C.c_longlong),
                ("max_rel_residual", C.c_double * 2), ("t_coarse_ms", C.c_double), ("t_fine_ms", C.c_double),
                ("n_systems", C.c_longlong * 2), ("n_rows", C.c_longlong * 2), ("nnz", C.c_longlong * 2),
                ("fine_dofs", C.c_longlong), ("kernel_launches", C.c_longlong),
                ("t_krylov_ms", C.c_double * 2), ("bytes_krylov", C.c_double * 2),
                ("krylov_launches", C.c_longlong * 2), ("coarse_factorizations", C.c_longlong),
                ("t_coarse_part_ms", C.c_double * 3), ("h2d_bytes", C.c_longlong), ("d2h_bytes", C.c_longlong)]


class LPFEMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")


_LIB = None


def lib() -> C.CDLL:
    """Load liblpfem.so (raises if it was not built: there is no fallback path)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2311_05170_b200.build` (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.lpfem_create.argtypes = [P(Geometry), P(Coeffs), P(Data), C.c_double, C.c_double, C.c_double,
                                   P(C.c_int), P(Opts), P(Dist), P(C.c_void_p)]
        L.lpfem_step.argtypes = [C.c_void_p, C.c_double]
        L.lpfem_step_group.argtypes = [P(C.c_void_p), C.c_int, C.c_double]
        L.lpfem_inject_fault.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.lpfem_placement.argtypes = [C.c_int, P(C.c_int), P(C.c_int), P(C.c_int), C.c_int, C.c_int, C.c_void_p]
        L.lpfem_get_sizes.argtypes = [C.c_void_p, P(C.c_longlong), P(C.c_longlong)]
        L.lpfem_get_fields.argtypes = [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int, C.c_int]
        L.lpfem_get_coarse_fields.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        L.lpfem_get_mesh.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, P(C.c_longlong)]
        L.lpfem_get_layout.argtypes = [C.c_void_p] + [C.c_void_p] * 6 + [P(C.c_int)]
        L.lpfem_get_stats.argtypes = [C.c_void_p, P(Stats)]
        L.lpfem_bench_spmv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, P(C.c_double), P(C.c_double)]
        L.lpfem_get_system.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, P(C.c_longlong), P(C.c_longlong),
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.lpfem_last_error.argtypes = [C.c_void_p]
        L.lpfem_last_error.restype = C.c_char_p
        L.lpfem_status_string.argtypes = [C.c_int]
        L.lpfem_status_string.restype = C.c_char_p
        L.lpfem_destroy.argtypes = [C.c_void_p]
        L.lpfem_nccl_unique_id.argtypes = [C.c_void_p]
        L.lpfem_halo_plan.argtypes = [C.c_int, P(C.c_int), P(C.c_int), P(C.c_int), C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, P(C.c_longlong)]
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


class LPFEM:
    """One context (one GPU, one rank).  cfg: a dict from ``lpfem_inputs.config``."""

    def __init__(self, cfg: dict, rank: int = 0, world: int = 1, device: int = 0, stream: int | None = None,
                 nccl_id: bytes | None = None, max_iter: int = 20000, transport: str = "nccl",
                 world_invariant: bool = False):
        L = lib()
        d = cfg["dim"]
        g = Geometry(dim=d)
        for a in range(d):
            g.porous_lo[a], g.porous_hi[a] = cfg["porous_lo"][a], cfg["porous_hi"][a]
            g.conduit_lo[a], g.conduit_hi[a] = cfg["conduit_lo"][a], cfg["conduit_hi"][a]
        co = cfg["coeffs"]
        c = Coeffs()
        for i in range(3):
            c.phi[i], c.C[i], c.k[i] = co["phi"][i], co["C"][i], co["k"][i]
        for k in ("sigma", "sigma_star", "mu_tilde", "nu", "rho", "alpha", "eta"):
            setattr(c, k, co[k])
        self._kmult = None
        if cfg.get("k_mult") is not None:
            self._kmult = np.ascontiguousarray(cfg["k_mult"], dtype=np.float64)
            c.k_mult = self._kmult.ctypes.data_as(C.POINTER(C.c_double))
        dat = Data(problem=PROB[cfg["problem"]], inflow_peak=cfg.get("inflow_peak", 1.0),
                   const_value=cfg.get("const_value", 1.0))
        o = Opts(lag_mode=LAG[cfg.get("lag_mode", "composite")], krylov_rtol=cfg.get("krylov_rtol", 1e-12),
                 max_iter=max_iter, gmres_restart=0, picard_rtol=cfg.get("picard_rtol", 1e-13),
                 picard_max=cfg.get("picard_max", 50), world_invariant=int(world_invariant),
                 algorithm=int(cfg.get("algorithm", 3)))
        ds = Dist(rank=rank, world=world, device=device, cuda_stream=stream, transport=TRANSPORT[transport])
        if nccl_id is not None:
            C.memmove(ds.nccl_id, nccl_id, 128)
        grid = (C.c_int * 3)(*(list(cfg["grid"]) + [1] * (3 - d)))
        h = C.c_void_p()
        self.cfg = cfg
        self.d = d
        st = L.lpfem_create(C.byref(g), C.byref(c), C.byref(dat), cfg["H"], cfg["h"], cfg["overlap"], grid,
                            C.byref(o), C.byref(ds), C.byref(h))
        if st != 0:
            raise LPFEMError(st, "lpfem_create failed")
        self._h = h
        n2 = (C.c_longlong * 2)()
        n1 = (C.c_longlong * 2)()
        L.lpfem_get_sizes(self._h, n2, n1)
        self.n_p2 = (n2[0], n2[1])
        self.n_p1 = n1[1]

    def _check(self, st: int):
        if st != 0:
            raise LPFEMError(st, lib().lpfem_last_error(self._h).decode())

    def step(self, dt: float | None = None):
        self._check(lib().lpfem_step(self._h, self.cfg["dt"] if dt is None else dt))

    def inject_fault(self, family: int, max_iter: int):
        """Test hook (lpfem_inject_fault): cap the fine Krylov iterations of family 0 (porous) / 1 (conduit)."""
        self._check(lib().lpfem_inject_fault(self._h, family, max_iter))

    def fields(self) -> dict:
        """Composite fine fields at t_n as host numpy arrays (global lexicographic, x fastest)."""
        np2p, np2c = self.n_p2
        out = {k: np.empty(np2p) for k in ("pF", "pf", "pm")}
        out["u"] = np.empty((self.d, np2c))
        out["p"] = np.empty(self.n_p1)
        self._check(lib().lpfem_get_fields(self._h, _ptr(out["pF"]), _ptr(out["pf"]), _ptr(out["pm"]),
                                           _ptr(out["u"]), _ptr(out["p"]), 0, 0))
        return out

    def fields_into(self, pF, pf, pm, u, p, on_device: bool = True):
        """Copy into caller buffers given as raw pointers (e.g. torch tensors' data_ptr())."""
        self._check(lib().lpfem_get_fields(self._h, C.c_void_p(pF), C.c_void_p(pf), C.c_void_p(pm), C.c_void_p(u),
                                           C.c_void_p(p), 1 if on_device else 0, 0))

    def coarse_fields(self) -> dict:
        d = self.d
        nc = [int(round((self.cfg["porous_hi"][a] - self.cfg["porous_lo"][a]) / self.cfg["H"])) for a in range(d)]
        ncc = [int(round((self.cfg["conduit_hi"][a] - self.cfg["conduit_lo"][a]) / self.cfg["H"])) for a in range(d)]
        n2p = int(np.prod([2 * k + 1 for k in nc]))
        n2c = int(np.prod([2 * k + 1 for k in ncc]))
        n1c = int(np.prod([k + 1 for k in ncc]))
        out = {k: np.empty(n2p) for k in ("pF", "pf", "pm")}
        out["u"] = np.empty((d, n2c))
        out["p"] = np.empty(n1c)
        self._check(lib().lpfem_get_coarse_fields(self._h, _ptr(out["pF"]), _ptr(out["pf"]), _ptr(out["pm"]),
                                                  _ptr(out["u"]), _ptr(out["p"])))
        return out

    def mesh(self, which: int):
        n = (C.c_longlong * 2)()
        self._check(lib().lpfem_get_mesh(self._h, which, None, None, n))
        coords = np.empty((n[0], self.d))
        cells = np.empty((n[1], (self.d + 1) * (self.d + 2) // 2), dtype=np.int32)
        self._check(lib().lpfem_get_mesh(self._h, which, _ptr(coords), _ptr(cells), n))
        return coords, cells

    def layout(self) -> list[dict]:
        nmax = 2 * int(np.prod(self.cfg["grid"]))
        reg = np.zeros(nmax, np.int32)
        pos = np.zeros(nmax, np.int32)
        arrs = [np.zeros(3 * nmax, np.int32) for _ in range(4)]
        n = C.c_int()
        self._check(lib().lpfem_get_layout(self._h, _ptr(reg), _ptr(pos), *[_ptr(a) for a in arrs], C.byref(n)))
        out = []
        for i in range(n.value):
            out.append({"region": "pc"[reg[i]], "pos": int(pos[i]),
                        "core0": tuple(arrs[0][3 * i:3 * i + self.d]), "core1": tuple(arrs[1][3 * i:3 * i + self.d]),
                        "box0": tuple(arrs[2][3 * i:3 * i + self.d]), "box1": tuple(arrs[3][3 * i:3 * i + self.d])})
        return out

    def bench_spmv(self, family: int = 1, reps: int = 10, flush: bool = True) -> dict:
        """lpfem_bench_spmv: mean device ms and algorithmic bytes of one batched SpMV over a family."""
        ms, b = C.c_double(), C.c_double()
        self._check(lib().lpfem_bench_spmv(self._h, family, reps, int(flush), C.byref(ms), C.byref(b)))
        return {"ms": ms.value, "bytes": b.value, "gbs": b.value / (ms.value * 1e-3) / 1e9}

    def stats(self) -> dict:
        s = Stats()
        self._check(lib().lpfem_get_stats(self._h, C.byref(s)))
        out = {}
        for name, _ in Stats._fields_:
            v = getattr(s, name)
            out[name] = list(v) if hasattr(v, "__len__") else v
        return out

    def system(self, family: int, index: int, field: int = 0) -> dict:
        nr, nz = C.c_longlong(), C.c_longlong()
        L = lib()
        self._check(L.lpfem_get_system(self._h, family, index, field, C.byref(nr), C.byref(nz), None, None, None, None,
                                       None))
        rp = np.empty(nr.value + 1, np.int64)
        col = np.empty(nz.value, np.int32)
        val = np.empty(nz.value)
        rhs = np.empty(nr.value)
        x = np.empty(nr.value)
        self._check(L.lpfem_get_system(self._h, family, index, field, C.byref(nr), C.byref(nz), _ptr(rp), _ptr(col),
                                       _ptr(val), _ptr(rhs), _ptr(x)))
        return {"rowptr": rp, "col": col, "val": val, "rhs": rhs, "x": x}

    def close(self):
        if getattr(self, "_h", None):
            lib().lpfem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    st = lib().lpfem_nccl_unique_id(buf)
    if st != 0:
        raise LPFEMError(st, "ncclGetUniqueId failed")
    return bytes(buf)


def _i3(v, dim):
    return (C.c_int * 3)(*(list(v) + [1] * (3 - dim)))


def placement(dim: int, n_cells_p, n_cells_c, grid, overlap_cells: int, world: int) -> np.ndarray:
    """lpfem_placement: rank of every subdomain position (LPT on box cells, csrc/halo.h)."""
    out = np.empty(int(np.prod(grid)), np.int32)
    st = lib().lpfem_placement(dim, _i3(n_cells_p, dim), _i3(n_cells_c, dim), _i3(grid, dim), overlap_cells, world,
                               _ptr(out))
    if st != 0:
        raise LPFEMError(st, "lpfem_placement")
    return out


def halo_plan(dim: int, n_cells, grid, overlap_cells: int, rank: int, world: int, kind: str, peer: int,
              vertex_only: bool = False, region: int = 0, n_cells_other=None) -> np.ndarray:
    """Host-side multi-GPU plan (lpfem_halo_plan) of one region: kind "need" | "give" | "owned".  n_cells: the
    region's fine cells per axis; n_cells_other: the other region's (default: the same)."""
    L = lib()
    k = {"need": 0, "give": 1, "owned": 2}[kind]
    other = n_cells if n_cells_other is None else n_cells_other
    ncp, ncc = (n_cells, other) if region == 0 else (other, n_cells)
    args = (dim, _i3(ncp, dim), _i3(ncc, dim), _i3(grid, dim), overlap_cells, region, rank, world, int(vertex_only),
            k, peer)
    n = C.c_longlong()
    st = L.lpfem_halo_plan(*args, None, C.byref(n))
    if st != 0:
        raise LPFEMError(st, "lpfem_halo_plan")
    out = np.empty(n.value, np.int32)
    L.lpfem_halo_plan(*args, _ptr(out), C.byref(n))
    return out


class LocalGroup:
    """All `world` ranks of the multi-rank path as contexts of THIS process (LPFEM_TRANSPORT_LOCAL), stepped
    together by lpfem_step_group: same placement, halo plan, pack/unpack and gather code as the NCCL transport,
    runnable on one GPU (tests).  fields() gathers on rank 0."""

    _next_key = 0

    def __init__(self, cfg: dict, world: int, device: int = 0, world_invariant: bool = False, **kw):
        LocalGroup._next_key += 1
        key = f"lpfem-local-{os.getpid()}-{LocalGroup._next_key}".encode().ljust(128, b"\0")
        self.cfg = cfg
        self.ranks = [LPFEM(cfg, rank=r, world=world, device=device, nccl_id=key, transport="local",
                            world_invariant=world_invariant, **kw) for r in range(world)]

    def step(self, dt: float | None = None):
        arr = (C.c_void_p * len(self.ranks))(*[r._h.value for r in self.ranks])
        st = lib().lpfem_step_group(arr, len(self.ranks), self.cfg["dt"] if dt is None else dt)
        if st != 0:
            raise LPFEMError(st, lib().lpfem_last_error(self.ranks[0]._h).decode())

    def fields(self) -> dict:
        return self.ranks[0].fields()

    def stats(self) -> list:
        return [r.stats() for r in self.ranks]

    def close(self):
        for r in self.ranks:
            r.close()
