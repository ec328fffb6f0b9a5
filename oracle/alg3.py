"""Algorithm 3, local parallel finite element algorithm (oracle; test infrastructure).

Paper: Algorithm 3.
  Step 1  coarse decoupled marching on T_H       -> alg1.Alg1 on (H) grids
  Step 2  overlapping subdomains D_j subset Omega_j -> mesh.subdomains
  Step 3  local fine corrections:
          porous eqs. pFlocalFully, pflocalFully, pmlocalFully,
          conduit eq. uclocalFully               -> Alg3._porous / Alg3._conduit
  Step 4  correction of data on the cores D_j    -> write-back by owner (C3)

Each local problem is written in the paper's correction form: unknown e, with
the bracketed coarse residual on the right-hand side, solved by SuperLU
(scipy.sparse.linalg.splu).  Readings: C2 lag source (mode "composite" = B,
"subdomain" = A), C4/C5 boundary data of e, C6 mean-zero multiplier on enclosed
conduit subdomains (only with the pressure_art = "free" flag; default C4 fixes delta = 0 on the
artificial faces), C10 plain convection, C12 initial data by interpolation,
C13 loads M I_h q, C14 typo fixes, C18 t_{n+1} = (n+1) dt.
"""
from __future__ import annotations

import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import mesh as M
from .alg1 import ORDER_SADDLE, ORDER_SPD, PIVOT, Alg1, PorousOps, make_conduit_ops, saddle
from .fem import prolongation
from .mms import Problem

FIELDS = ("pF", "pf", "pm")


class DirichletLU:
    """LU of A restricted to the free dofs, reused for many right-hand sides (porous: time-invariant)."""

    def __init__(self, A: sp.csr_matrix, fixed: np.ndarray, border: np.ndarray | None = None, spd: bool = True):
        self.fixed = fixed
        self.free = free = ~fixed
        Aff = A[free][:, free]
        self.Afd = A[free][:, fixed]
        self.n = Aff.shape[0]
        self.border = border is not None
        if self.border:
            m = border[free]
            Aff = sp.bmat([[Aff, sp.csr_matrix(m[:, None])], [sp.csr_matrix(m[None, :]), None]])
        order = ORDER_SPD if spd and border is None else ORDER_SADDLE
        self.lu = spla.splu(Aff.tocsc(), permc_spec=order, diag_pivot_thresh=PIVOT[order])
        self.Aff = Aff.tocsr()

    def solve(self, b: np.ndarray, vals: np.ndarray):
        x = np.zeros(len(self.fixed))
        x[self.fixed] = vals
        rhs = b[self.free] - self.Afd @ vals
        if self.border:
            rhs = np.concatenate([rhs, [0.0]])
        sol = self.lu.solve(rhs)
        self.last_rel_residual = np.linalg.norm(self.Aff @ sol - rhs) / max(np.linalg.norm(rhs), 1e-300)
        x[self.free] = sol[: self.n]
        return x


class Alg3:
    def __init__(self, cfg: dict, positions=None, regions=("p", "c")):
        """positions: optional list of subdomain positions (lexicographic grid index) to set up and solve
        (sampled parity at full size); regions: which regions' subdomains to set up.  Construction only: the
        arithmetic of every solved subdomain is unchanged."""
        self.cfg = cfg
        self.d = d = cfg["dim"]
        self.prob = Problem(cfg)
        self.Gp, self.Gc = M.region_grids(cfg, "h")
        self.GpH, self.GcH = M.region_grids(cfg, "H")
        self.R = R = int(round(cfg["H"] / cfg["h"]))
        ov = int(round(cfg["overlap"] / cfg["h"]))
        self.mode = cfg.get("lag_mode", "composite")
        self.coarse = Alg1(cfg, self.GpH, self.GcH, 1, self.prob)
        self.grid_m = tuple(cfg["grid"])
        self.sub_p = M.subdomains(self.Gp, self.grid_m, ov)
        self.sub_c = M.subdomains(self.Gc, self.grid_m, ov)
        if positions is not None:
            keep = set(int(q) for q in positions)
            lexpos = lambda sub: int(M.lex_index(np.asarray(sub.index), np.zeros(d, np.int64), np.asarray(self.grid_m)))
            self.sub_p = [sb for sb in self.sub_p if lexpos(sb) in keep]
            self.sub_c = [sb for sb in self.sub_c if lexpos(sb) in keep]
        if "p" not in regions:
            self.sub_p = []
        if "c" not in regions:
            self.sub_c = []
        # global fine node sets
        self.box_p = M.Box(self.Gp, (0,) * d, self.Gp.n)
        self.box_c = M.Box(self.Gc, (0,) * d, self.Gc.n)
        self.Xp = self.Gp.coords(self.box_p.node_g)
        self.Xc = self.Gc.coords(self.box_c.node_g)
        self.Xc1 = self.Gc.coords(self.box_c.vert_g)
        pr = self.prob
        # C12: composite u^h_0 = I_h u_0
        self.comp = {f: pr.porous(f, self.Xp, 0.0) for f in FIELDS}
        top = self.box_c.node_g[:, -1] == 2 * self.Gc.n[-1]
        self.comp["u"] = pr.velocity(self.Xc, 0.0, top) if pr.kind == "mms" else np.zeros((d, len(self.Xc)))
        self.comp["p"] = pr.pressure(self.Xc1, 0.0)
        self.t_index = 0
        self.timing = {"coarse": 0.0, "fine": 0.0}
        t0 = time.perf_counter()
        self.P = [self._setup_porous(s) for s in self.sub_p]
        self.C = [self._setup_conduit(s) for s in self.sub_c]
        self.timing["setup"] = time.perf_counter() - t0
        # C12: e_j^0 = (I_h u_0 - P I_H u_0) on the box (mode A state)
        cs = self.coarse.state
        for P in self.P:
            P["e"] = {f: self.comp[f][P["gidx"]] - P["Pr"] @ cs[f] for f in FIELDS}
        for C in self.C:
            C["e"] = self.comp["u"][:, C["gidx"]] - np.stack([C["Pr2"] @ cs["u"][a] for a in range(d)])

    # ------------------------------------------------------------------ setup
    def _setup_porous(self, sub: M.Subdomain) -> dict:
        box = sub.box
        ops = PorousOps(self.cfg, box, self.R)
        cls = box.classes()
        fixed = cls >= M.ART
        gidx = self.box_p.p2_index(box.node_g)
        own = M.owner(box.node_g, self.Gp, self.grid_m) == M.lex_index(np.asarray(sub.index), np.zeros(self.d, np.int64), np.asarray(self.grid_m))
        Pr = prolongation(self.GpH, box.node_g, self.R, 2)
        # coarse conduit velocity at the box's Gamma nodes (flux term)
        gam = np.nonzero(box.node_g[:, -1] == self.Gp.gamma_g)[0]
        gc = box.node_g[gam].copy()
        gc[:, -1] = self.Gc.gamma_g
        Pu = prolongation(self.GcH, gc, self.R, 2) if len(gam) else None
        lu = {f: DirichletLU(ops.A[f], fixed) for f in FIELDS}
        return {"sub": sub, "ops": ops, "cls": cls, "fixed": fixed, "gidx": gidx, "own": own, "Pr": Pr,
                "gam": gam, "Pu": Pu, "lu": lu, "X": self.Gp.coords(box.node_g)}

    def _setup_conduit(self, sub: M.Subdomain) -> dict:
        box, d = sub.box, self.d
        ops = make_conduit_ops(self.cfg, box, self.R)
        cls = box.classes()
        n2, n1 = box.node_g.shape[0], box.vert_g.shape[0]
        fixed_v = np.concatenate([cls >= M.ART] * d)
        # C4: the pressure correction lives in Q_0^h(Omega_j) (compact support): delta = 0 on the
        # closure of the artificial faces.  Flag pressure_art = "free": delta free there (+ C6 multiplier).
        p_free_art = self.cfg.get("pressure_art", "zero") == "free"
        fixed_p = np.zeros(n1, bool) if p_free_art else box.on_artificial(box.vert_g)
        fixed = np.concatenate([fixed_v, fixed_p])
        gidx = self.box_c.p2_index(box.node_g)
        gidx1 = self.box_c.p1_index(box.vert_g)
        sidx = M.lex_index(np.asarray(sub.index), np.zeros(d, np.int64), np.asarray(self.grid_m))
        own = M.owner(box.node_g, self.Gc, self.grid_m) == sidx
        own1 = M.owner(box.vert_g, self.Gc, self.grid_m) == sidx
        Pr2 = prolongation(self.GcH, box.node_g, self.R, 2)
        Pr1 = prolongation(self.GcH, box.vert_g, self.R, 1)
        gam = np.nonzero(box.node_g[:, -1] == self.Gc.gamma_g)[0]
        gp = box.node_g[gam].copy()
        gp[:, -1] = self.Gp.gamma_g
        PpF = prolongation(self.GpH, gp, self.R, 2) if len(gam) else None
        border = None
        if p_free_art and sub.enclosed and self.cfg.get("pressure_constraint", "mean_zero") == "mean_zero":
            border = np.concatenate([np.zeros(d * n2), ops.fem.p1_mass_vector()])
        top = box.node_g[:, -1] == 2 * self.Gc.n[-1]
        return {"sub": sub, "ops": ops, "cls": cls, "fixed": fixed, "gidx": gidx, "gidx1": gidx1, "own": own,
                "own1": own1, "Pr2": Pr2, "Pr1": Pr1, "gam": gam, "PpF": PpF, "border": border,
                "X": self.Gc.coords(box.node_g), "top": top, "Mv": ops.fem.vec_mass(1.0)}

    # ------------------------------------------------------------------ step
    def step(self):
        cfg, d, pr = self.cfg, self.d, self.prob
        t = (self.t_index + 1) * cfg["dt"]  # C18
        t0 = time.perf_counter()
        old = {k: np.copy(v) for k, v in self.coarse.state.items()}  # u_H^n
        self.coarse.step()  # Algorithm 3 Step 1
        new = self.coarse.state  # u_H^{n+1}
        t1 = time.perf_counter()
        comp_new = {k: np.copy(v) for k, v in self.comp.items()}
        for P in self.P:
            self._porous(P, old, new, t, comp_new)
        for C in self.C:
            self._conduit(C, old, new, t, comp_new)
        self.comp = comp_new
        self.t_index += 1
        t2 = time.perf_counter()
        self.timing["coarse"] += t1 - t0
        self.timing["fine"] += t2 - t1

    def _porous(self, P: dict, old: dict, new: dict, t: float, comp_new: dict):
        """Step 3(1): eqs. pFlocalFully, pflocalFully, pmlocalFully on Omega_pj."""
        ops, pr = P["ops"], self.prob
        Mm, c = ops.M, ops.c
        K = {"pF": ops.K[2], "pf": ops.K[1], "pm": ops.K[0]}
        PH1 = {f: P["Pr"] @ new[f] for f in FIELDS}  # P p_iH^{n+1}
        PH0 = {f: P["Pr"] @ old[f] for f in FIELDS}  # P p_iH^n
        if self.mode == "composite":  # C2 mode B: e~^n = u^h_n - P u_H^n on Omega_j
            en = {f: self.comp[f][P["gidx"]] - PH0[f] for f in FIELDS}
        else:  # mode A: the subdomain's own e_j^n (P:1279-1305 as printed)
            en = P["e"]
        X = P["X"]
        q = {f: Mm @ pr.q(f, X, t) for f in FIELDS}  # (q_i(t_{n+1}), v), C13
        # <u_cH^n . n_c, v_F>_{Gamma cap dOmega_pj}, n_c = -e_last
        flux = np.zeros(len(X))
        if P["Pu"] is not None:
            w = np.zeros(len(X))
            w[P["gam"]] = -(P["Pu"] @ old["u"][-1])
            flux = ops.MG @ w
        rhs = {
            "pF": c[2] * (Mm @ en["pF"]) + ops.M_Ff @ en["pf"] + q["pF"]
            - (c[2] * (Mm @ (PH1["pF"] - PH0["pF"])) + K["pF"] @ PH1["pF"] + ops.M_Ff @ (PH1["pF"] - PH0["pf"]))
            + flux,
            "pf": c[1] * (Mm @ en["pf"]) + ops.M_fm @ en["pm"] + ops.M_Ff @ en["pF"] + q["pf"]
            - (c[1] * (Mm @ (PH1["pf"] - PH0["pf"])) + K["pf"] @ PH1["pf"] + ops.M_fm @ (PH1["pf"] - PH0["pm"])
               + ops.M_Ff @ (PH1["pf"] - PH0["pF"])),
            "pm": c[0] * (Mm @ en["pm"]) + ops.M_fm @ en["pf"] + q["pm"]
            - (c[0] * (Mm @ (PH1["pm"] - PH0["pm"])) + K["pm"] @ PH1["pm"] + ops.M_fm @ (PH1["pm"] - PH0["pf"])),
        }
        fixed, cls = P["fixed"], P["cls"]
        dirm = cls[fixed] == M.DIR
        for f in FIELDS:
            vals = np.zeros(int(fixed.sum()))
            # C5: e = I_h g(t_{n+1}) - P p_H^{n+1} on dir nodes; C4: e = 0 on artificial nodes
            vals[dirm] = pr.porous(f, X[fixed][dirm], t) - PH1[f][fixed][dirm]
            e = P["lu"][f].solve(rhs[f], vals)
            P["e"][f] = e
            full = PH1[f] + e  # Step 4: p_iH^{n+1} + e_i
            comp_new[f][P["gidx"][P["own"]]] = full[P["own"]]

    def _conduit(self, C: dict, old: dict, new: dict, t: float, comp_new: dict):
        """Step 3(2): eq. uclocalFully on Omega_cj'."""
        ops, pr, d = C["ops"], self.prob, self.d
        eta = ops.eta
        n2 = C["X"].shape[0]
        U = np.stack([C["Pr2"] @ new["u"][a] for a in range(d)])  # u_cH^{n+1} on the fine box
        U0 = np.stack([C["Pr2"] @ old["u"][a] for a in range(d)])  # u_cH^n
        Ph = C["Pr1"] @ new["p"]  # p_H^{n+1} (P1)
        if self.mode == "composite":
            en = self.comp["u"][:, C["gidx"]] - U0
        else:
            en = C["e"]
        N_U = ops.fem.convection(U, eta)  # b_N(U, e, v)
        R_U = ops.fem.convection_reaction(U, eta)  # b_N(e, U, v)
        A_u = (ops.A_lin + N_U + R_U).tocsr()
        K = saddle(A_u, ops.Bdiv)
        f = pr.f(C["X"], t)
        Uf = U.ravel()
        bracket = ops.Mu @ (Uf - U0.ravel()) + (ops.Visc + ops.Fr) @ Uf - ops.Bdiv.T @ Ph + N_U @ Uf
        pFg = np.zeros(n2)
        if C["PpF"] is not None:
            pFg[C["gam"]] = C["PpF"] @ old["pF"]  # P p_FH^n on Gamma
        rhs_v = eta * (C["Mv"] @ f.ravel()) + ops.Mu @ en.ravel() - bracket + ops.gamma_load(pFg)
        rhs_p = -(ops.Bdiv @ Uf)  # -[ -b_eta(u_cH^{n+1}, q) ]
        b = np.concatenate([rhs_v, rhs_p])
        fixed, cls = C["fixed"], C["cls"]
        dirn = cls == M.DIR
        vals_full = np.zeros((d, n2))
        g = pr.velocity(C["X"][dirn], t, C["top"][dirn])
        vals_full[:, dirn] = g - U[:, dirn]  # C5
        vals = np.concatenate([vals_full[a][fixed[a * n2:(a + 1) * n2]] for a in range(d)]
                              + [np.zeros(int(fixed[d * n2:].sum()))])
        lu = DirichletLU(K, fixed, C["border"], spd=False)
        x = lu.solve(b, vals)
        C["last_rel_residual"] = lu.last_rel_residual
        e = x[: d * n2].reshape(d, n2)
        delta = x[d * n2:]
        C["e"] = e
        full_u = U + e  # Step 4
        full_p = Ph + delta
        comp_new["u"][:, C["gidx"][C["own"]]] = full_u[:, C["own"]]
        comp_new["p"][C["gidx1"][C["own1"]]] = full_p[C["own1"]]

    # ------------------------------------------------------------------ output
    def fields(self) -> dict:
        return {k: np.copy(v) for k, v in self.comp.items()}


def run(cfg: dict, steps: int | None = None) -> list[dict]:
    """Fields after each step (list index n-1 = t_n)."""
    a = Alg3(cfg)
    out = []
    for _ in range(cfg["steps"] if steps is None else steps):
        a.step()
        out.append(a.fields())
    return out
