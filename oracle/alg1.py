"""Algorithm 1, partitioned time stepping on one mesh (oracle; test infrastructure).

Paper: Algorithm 1, eqs. fullypF, fullypf, fullypm (porous, BE with
lagged partners and lagged flux u^n) and fullyuc (implicit NS with lagged p_F^n).
Algorithm 3 Step 1 (eqs. pFFully..pcFully) is exactly this scheme
on T_H; the nonlinear NS step is solved by Picard from u^n (reading C11).

Also provides the porous / conduit operator assembly reused by alg3.py:
  A_F = c_F M + K[k_F/mu] + M[sigma* k_f/mu]
  A_f = c_f M + K[k_f/mu] + M[sigma k_m/mu + sigma* k_f/mu]
  A_m = c_m M + K[k_m/mu] + M[sigma k_m/mu]          (c_i = phi_i C_i / dt)
with the permeabilities scaled per porous coarse cell by k_mult (C15).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import mesh as M
from .fem import BoxFEM
from .mms import Problem

IDX = {"pm": 0, "pf": 1, "pF": 2}


def coarse_cell_mult(cfg: dict, cells: np.ndarray, ratio: int) -> np.ndarray:
    """Multiplier s of the porous coarse cell containing each cell (cells in a mesh `ratio` times finer than T_H)."""
    if cfg.get("k_mult") is None:
        return np.ones(len(cells))
    d = cfg["dim"]
    nH = [int(round((cfg["porous_hi"][a] - cfg["porous_lo"][a]) / cfg["H"])) for a in range(d)]
    cH = np.asarray(cells) // ratio
    return np.asarray(cfg["k_mult"])[M.lex_index(cH, np.zeros(d, np.int64), np.asarray(nH))]


# Fill-reducing column orderings for SuperLU (no arithmetic difference: the LU solves the same system).
# SPD porous systems: minimum degree on A^T + A with diagonal pivots (no pivoting is needed for SPD matrices;
# 6x faster on a 3D 18^3 P2 box).  Saddle-point systems (zero pressure diagonal, so SuperLU pivots off the
# diagonal): minimum degree on A^T A, ~100x faster than A^T + A on a 64^2 Taylor-Hood box.
ORDER_SPD = "MMD_AT_PLUS_A"
ORDER_SADDLE = "MMD_ATA"
PIVOT = {ORDER_SPD: 0.0, ORDER_SADDLE: 1.0}


def solve_dirichlet(A: sp.csr_matrix, b: np.ndarray, fixed: np.ndarray, vals: np.ndarray, border=None,
                    spd: bool = True):
    """Solve A x = b with x[fixed] = vals (rows of fixed dofs dropped, columns moved to the RHS).
    border: optional dense column/row m over the free dofs (bordered Lagrange multiplier, C6)."""
    order = ORDER_SPD if spd else ORDER_SADDLE
    free = ~fixed
    x = np.zeros(A.shape[0])
    x[fixed] = vals
    Aff = A[free][:, free]
    rhs = b[free] - A[free][:, fixed] @ vals
    if border is not None:
        m = border[free]
        n = Aff.shape[0]
        Aff = sp.bmat([[Aff, sp.csr_matrix(m[:, None])], [sp.csr_matrix(m[None, :]), None]]).tocsc()
        rhs = np.concatenate([rhs, [0.0]])
        sol = spla.splu(Aff.tocsc(), permc_spec=order, diag_pivot_thresh=PIVOT[order]).solve(rhs)
        x[free] = sol[:n]
        return x
    x[free] = spla.splu(Aff.tocsc(), permc_spec=order, diag_pivot_thresh=PIVOT[order]).solve(rhs)
    return x


class PorousOps:
    """Porous operators of one box (fine subdomain or whole coarse region)."""

    def __init__(self, cfg: dict, box: M.Box, ratio: int):
        co = cfg["coeffs"]
        self.fem = fem = BoxFEM(box)
        s = coarse_cell_mult(cfg, fem.cell, ratio)
        mu = co["mu_tilde"]
        k = [co["k"][i] * s for i in range(3)]
        dt = cfg["dt"]
        c = [co["phi"][i] * co["C"][i] / dt for i in range(3)]
        self.M = fem.mass()
        self.K = [fem.stiffness(k[i] / mu) for i in range(3)]
        self.M_Ff = fem.mass(co["sigma_star"] * k[1] / mu)
        self.M_fm = fem.mass(co["sigma"] * k[0] / mu)
        self.c = c
        self.A = {
            "pF": (c[2] * self.M + self.K[2] + self.M_Ff).tocsr(),
            "pf": (c[1] * self.M + self.K[1] + self.M_fm + self.M_Ff).tocsr(),
            "pm": (c[0] * self.M + self.K[0] + self.M_fm).tocsr(),
        }
        self.MG = fem.facet_mass()  # int_Gamma phi_i phi_j


class ConduitOps:
    """Conduit operators of one box: (eta/dt) velocity mass, 2 nu eta (D,D), Gamma friction, divergence,
    Gamma loads.  Built by make_conduit_ops."""

    def gamma_load(self, pF_gamma: np.ndarray) -> np.ndarray:
        """-(eta/rho)<pF, v.n_c> - (eta nu alpha sqrt(kF)/mu)<grad_tau pF, P_tau v> with n_c = -e_last
        (P:1262-1264): the (d*n2,) load for pF given at the box's P2 nodes (only Gamma values matter)."""
        d, n2 = self.d, self.fem.n2
        out = np.zeros(d * n2)
        if self.MG_n is None:
            return out
        out[(d - 1) * n2:] += self.MG_n @ pF_gamma  # v.n_c = -v_last
        for a in range(d - 1):
            out[a * n2:(a + 1) * n2] -= self.TG[a] @ pF_gamma
        return out


def _facet_mult_for(cfg: dict, fem: BoxFEM, ratio_to_H: int) -> np.ndarray:
    """Multiplier of the porous coarse cell under each Gamma facet of a conduit box."""
    if fem.facets is None or cfg.get("k_mult") is None:
        return np.ones(0 if fem.facets is None else len(fem.facets["vol"]))
    d = cfg["dim"]
    nH = [int(round((cfg["porous_hi"][a] - cfg["porous_lo"][a]) / cfg["H"])) for a in range(d)]
    fc = fem.facets["cell"] // ratio_to_H  # tangential coarse cell
    cells = np.concatenate([fc, np.full((len(fc), 1), nH[-1] - 1)], axis=1)
    return np.asarray(cfg["k_mult"])[M.lex_index(cells, np.zeros(d, np.int64), np.asarray(nH))]


def make_conduit_ops(cfg: dict, box: M.Box, ratio_to_H: int) -> ConduitOps:
    ops = ConduitOps.__new__(ConduitOps)
    co = cfg["coeffs"]
    ops.cfg = cfg
    ops.d = d = box.d
    ops.fem = fem = BoxFEM(box)
    eta, nu, alpha = co["eta"], co["nu"], co["alpha"]
    ops.eta = eta
    ops.Mu = fem.vec_mass(eta / cfg["dt"])
    ops.Visc = fem.deformation(nu * eta)
    n2 = fem.n2
    if fem.facets is not None:
        kF = co["k"][2] * _facet_mult_for(cfg, fem, ratio_to_H)
        fric = eta * nu * alpha / np.sqrt(kF)  # eta nu alpha sqrt(d)/sqrt(tr Pi), Pi = k_F I
        ct = eta * nu * alpha * np.sqrt(kF) / co["mu_tilde"]
        ops.Fr = sp.block_diag([fem.facet_mass(fric) if a < d - 1 else sp.csr_matrix((n2, n2)) for a in range(d)]).tocsr()
        ops.MG_n = fem.facet_mass(None) * (eta / co["rho"])
        ops.TG = [fem.facet_tangential_grad(a, ct) for a in range(d - 1)]
    else:
        ops.Fr = sp.csr_matrix((d * n2, d * n2))
        ops.MG_n = None
        ops.TG = None
    ops.Bdiv = fem.divergence(eta)
    ops.A_lin = (ops.Mu + ops.Visc + ops.Fr).tocsr()
    return ops


def saddle(A_u: sp.csr_matrix, Bdiv: sp.csr_matrix) -> sp.csr_matrix:
    """[[A_u, -Bdiv^T], [Bdiv, 0]]: b_eta(v, p) = -eta (p, div v) in the momentum rows, -b_eta(u, q) = eta (q, div u)
    in the continuity rows."""
    return sp.bmat([[A_u, -Bdiv.T], [Bdiv, None]]).tocsr()


class Alg1:
    """Algorithm 1 on the meshes (Gp, Gc) of both regions; state at t_n."""

    def __init__(self, cfg: dict, Gp: M.Grid, Gc: M.Grid, ratio_to_H: int, prob: Problem | None = None):
        self.cfg, self.Gp, self.Gc = cfg, Gp, Gc
        self.d = cfg["dim"]
        self.prob = prob or Problem(cfg)
        self.box_p = M.Box(Gp, (0,) * self.d, Gp.n)
        self.box_c = M.Box(Gc, (0,) * self.d, Gc.n)
        self.por = PorousOps(cfg, self.box_p, ratio_to_H)
        self.con = make_conduit_ops(cfg, self.box_c, ratio_to_H)
        self.cls_p = self.box_p.classes(whole_region=True)
        self.cls_c = self.box_c.classes(whole_region=True)
        self.Xp = Gp.coords(self.box_p.node_g)
        self.Xc = Gc.coords(self.box_c.node_g)
        self.Xc1 = Gc.coords(self.box_c.vert_g)
        self.top_c = self.box_c.node_g[:, -1] == 2 * Gc.n[-1]
        # Gamma node maps between the regions (same tangential half-grid)
        gp = self.box_p.node_g
        self.gam_p = np.nonzero(gp[:, -1] == Gp.gamma_g)[0]
        gc_of_p = gp[self.gam_p].copy()
        gc_of_p[:, -1] = Gc.gamma_g
        self.gam_p_to_c = self.box_c.p2_index(gc_of_p)
        self.t_index = 0
        pr = self.prob
        self.state = {f: pr.porous(f, self.Xp, 0.0) for f in ("pF", "pf", "pm")}
        self.state["u"] = pr.velocity(self.Xc, 0.0, self.top_c) if pr.kind == "mms" else np.zeros((self.d, len(self.Xc)))
        self.state["p"] = pr.pressure(self.Xc1, 0.0)
        self.picard_rtol = cfg.get("picard_rtol", 1e-13)
        self.picard_max = cfg.get("picard_max", 50)
        self.picard_iters = []

    def flux_load(self, u: np.ndarray) -> np.ndarray:
        """int_Gamma (u . n_c) v_F, n_c = -e_last, as a vector over porous nodes."""
        w = np.zeros(self.box_p.node_g.shape[0])
        w[self.gam_p] = -u[-1][self.gam_p_to_c]
        return self.por.MG @ w

    def pF_on_conduit(self, pF: np.ndarray) -> np.ndarray:
        out = np.zeros(self.box_c.node_g.shape[0])
        out[self.gam_p_to_c] = pF[self.gam_p]
        return out

    def step(self):
        cfg, pr, d = self.cfg, self.prob, self.d
        n1 = self.t_index + 1
        t = n1 * cfg["dt"]  # C18
        S = self.state
        por = self.por
        fixed = self.cls_p == M.DIR
        q = {f: por.M @ pr.q(f, self.Xp, t) for f in ("pF", "pf", "pm")}
        c = por.c
        rhs = {
            "pF": c[2] * (por.M @ S["pF"]) + por.M_Ff @ S["pf"] + q["pF"] + self.flux_load(S["u"]),
            "pf": c[1] * (por.M @ S["pf"]) + por.M_fm @ S["pm"] + por.M_Ff @ S["pF"] + q["pf"],
            "pm": c[0] * (por.M @ S["pm"]) + por.M_fm @ S["pf"] + q["pm"],
        }
        new = {}
        for f in ("pF", "pf", "pm"):
            new[f] = solve_dirichlet(por.A[f], rhs[f], fixed, pr.porous(f, self.Xp[fixed], t))
        u_new, p_new = self.ns_step(S["u"], S["pF"], t)
        new["u"], new["p"] = u_new, p_new
        self.state = new
        self.t_index = n1

    def ns_step(self, u_n: np.ndarray, pF_n: np.ndarray, t: float):
        """eq. fullyuc / pcFully by Picard: wind w^0 = u^n (C11)."""
        con, pr, d = self.con, self.prob, self.d
        n2 = self.box_c.node_g.shape[0]
        n1 = self.box_c.vert_g.shape[0]
        eta = con.eta
        fixed_v = np.concatenate([self.cls_c == M.DIR] * d)
        fixed = np.concatenate([fixed_v, np.zeros(n1, bool)])
        g = pr.velocity(self.Xc[self.cls_c == M.DIR], t, self.top_c[self.cls_c == M.DIR])
        gvals = np.concatenate([g[a] for a in range(d)])
        f = pr.f(self.Xc, t)
        load = eta * (con.fem.vec_mass(1.0) @ f.ravel()) + con.Mu @ u_n.ravel() + con.gamma_load(self.pF_on_conduit(pF_n))
        b = np.concatenate([load, np.zeros(n1)])
        w = u_n.copy()
        for it in range(self.picard_max):
            A_u = con.A_lin + con.fem.convection(w, eta)
            x = solve_dirichlet(saddle(A_u, con.Bdiv), b, fixed, gvals, spd=False)
            u = x[: d * n2].reshape(d, n2)
            du = np.linalg.norm(u - w)
            w = u
            # C11: ||du||_2 <= rtol ||u||_2, or an absolute floor 1e-14 sqrt(N) for (near-)zero velocity
            if du <= self.picard_rtol * np.linalg.norm(u) or du <= 1e-14 * np.sqrt(u.size):
                self.picard_iters.append(it + 1)
                return u, x[d * n2:]
        raise RuntimeError("Picard did not converge (C11)")
