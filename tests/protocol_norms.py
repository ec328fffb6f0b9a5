"""Error norms of the paper's convergence study (test infrastructure, the norms of Tables 1-4).

The paper measures, at the final time, the piecewise H1 seminorm over the cores D_j,
|||e|||_1 = (sum_j |e_j|_{1,D_j}^2)^(1/2), and the piecewise L2 norm |||e|||_0.  The cores tile
the region, and on every core the composite field holds that subdomain's solution (Step 4 write-back,
P:1329-1337; a node on a core boundary carries its owner's value, reading C3), so the piecewise norms are
evaluated as integrals of the composite P2 field over the region's fine simplices (reading C28 in DESIGN.md).

Integrals: a Duffy-mapped Gauss-Legendre rule on every Kuhn triangle (exact for polynomials of degree
2 NQ - 2; the integrands here are smooth, the rule is taken fine enough that its error is far below the
discretisation error).  Exact values and gradients come from the manufactured solution's SymPy expressions
(oracle/mms.py, paper Ex1 P:1517-1521), differentiated symbolically.
"""
from __future__ import annotations

import itertools

import numpy as np
import sympy as S

from oracle import mesh as M

NQ = 6


def _rule(nq: int = NQ):
    g, w = np.polynomial.legendre.leggauss(nq)
    g, w = 0.5 * (g + 1.0), 0.5 * w
    u, v = np.meshgrid(g, g, indexing="ij")
    wu, wv = np.meshgrid(w, w, indexing="ij")
    l1 = u.ravel()
    l2 = (v * (1.0 - u)).ravel()
    lam = np.stack([1.0 - l1 - l2, l1, l2], axis=1)  # (Q, 3)
    wt = (wu * wv * (1.0 - u)).ravel() * 2.0          # sums to 1: integral over K = |K| sum wt f
    return lam, wt


def _p2_vals_grads(lam: np.ndarray):
    """P2 basis (vertices, then edges (0,1),(0,2),(1,2)) and d phi / d lambda_k at barycentric points (Q, 3)."""
    eds = list(itertools.combinations(range(3), 2))
    Q = lam.shape[0]
    phi = np.zeros((Q, 6))
    dphi = np.zeros((Q, 6, 3))
    for i in range(3):
        phi[:, i] = lam[:, i] * (2.0 * lam[:, i] - 1.0)
        dphi[:, i, i] = 4.0 * lam[:, i] - 1.0
    for k, (a, b) in enumerate(eds):
        phi[:, 3 + k] = 4.0 * lam[:, a] * lam[:, b]
        dphi[:, 3 + k, a] = 4.0 * lam[:, b]
        dphi[:, 3 + k, b] = 4.0 * lam[:, a]
    return phi, dphi


def region_geometry(grid: M.Grid):
    """Fine simplices of a whole 2D region: P2 node indices (E, 6), vertex coordinates (E, 3, 2)."""
    box = M.Box(grid, (0,) * grid.d, grid.n)
    p2, _p1, gv, _cell = box.simplices()
    X = grid.coords(gv.reshape(-1, grid.d)).reshape(gv.shape[0], 3, grid.d)
    return p2, X


def norms(grid: M.Grid, values: np.ndarray, exact, exact_grad, nq: int = NQ):
    """(L2 norm, H1 seminorm) of exact - u_h over the region, u_h the P2 field with nodal values `values`
    (global lexicographic); exact(X) -> (N,), exact_grad(X) -> (N, 2) at points X (N, 2)."""
    p2, X = region_geometry(grid)
    lam, wt = _rule(nq)
    phi, dphi = _p2_vals_grads(lam)
    J = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]], axis=2)   # (E, 2, 2): columns x1 - x0, x2 - x0
    area = 0.5 * np.abs(np.linalg.det(J))
    Jinv = np.linalg.inv(J)                                          # rows: grad lambda_1, grad lambda_2
    gl = np.concatenate([-(Jinv[:, 0:1] + Jinv[:, 1:2]), Jinv], axis=1)  # (E, 3, 2) grad lambda_k
    u = values[p2]                                                   # (E, 6)
    uh = u @ phi.T                                                   # (E, Q)
    duh = np.einsum("ei,qik,ekc->eqc", u, dphi, gl)                  # (E, Q, 2)
    P = np.einsum("qk,ekc->eqc", lam, X)                             # (E, Q, 2) points
    ex = exact(P.reshape(-1, 2)).reshape(uh.shape)
    dex = exact_grad(P.reshape(-1, 2)).reshape(duh.shape)
    l2 = np.sqrt(np.sum(area[:, None] * wt[None, :] * (ex - uh) ** 2))
    h1 = np.sqrt(np.sum(area[:, None] * wt[None, :] * np.sum((dex - duh) ** 2, axis=2)))
    return l2, h1


def ex1_functions(t: float):
    """Exact value / gradient callables of paper Ex1 at time t, from oracle/mms.py's expressions."""
    from oracle.mms import _ex1_symbols
    (x, y), ts, sol = _ex1_symbols()
    out = {}
    for k in ("pF", "pf", "pm", "p"):
        e = sol[k].subs(ts, t)
        out[k] = _pair(e, x, y)
    for a in range(2):
        out[f"u{a}"] = _pair(sol["u"][a].subs(ts, t), x, y)
    return out


def _pair(e, x, y):
    f = S.lambdify((x, y), e, "numpy")
    gx = S.lambdify((x, y), S.diff(e, x), "numpy")
    gy = S.lambdify((x, y), S.diff(e, y), "numpy")

    def val(P):
        return np.broadcast_to(np.asarray(f(P[:, 0], P[:, 1]), dtype=float), P.shape[:1]).copy()

    def grad(P):
        a = np.broadcast_to(np.asarray(gx(P[:, 0], P[:, 1]), dtype=float), P.shape[:1])
        b = np.broadcast_to(np.asarray(gy(P[:, 0], P[:, 1]), dtype=float), P.shape[:1])
        return np.stack([a, b], axis=1)

    return val, grad


def protocol_config(level: int, algorithm: int = 3) -> dict:
    """Paper Ex1 protocol: all coefficients 1, 2x2 subdomains per region with the fixed extension
    1/4, h = H^2, dt = h^2, T = 1; level 0, 1, 2 -> h = 1/4, 1/16, 1/64 (H = 1/2, 1/4, 1/8).  Taylor-Hood P2-P1
    and P2 porous pressures (reading C1) instead of the paper's MINI / P1."""
    import lpfem_inputs as I
    H = 0.5 ** (level + 1)
    h = H * H
    dt = h * h
    steps = int(round(1.0 / dt))
    co = dict(I.BASE_COEFFS)
    co["k"] = [1.0, 1.0, 1.0]
    if algorithm == 1:
        return I.make_config(dim=2, H=H, h=h, grid=1, dt=dt, steps=steps, problem="mms", overlap=0.0,
                             algorithm=1, coeffs=co, name=f"protocol{level}_alg1")
    return I.make_config(dim=2, H=H, h=h, grid=2, dt=dt, steps=steps, problem="mms", overlap=0.25, coeffs=co,
                         name=f"protocol{level}")


def table_errors(cfg: dict, fields: dict) -> dict:
    """The columns of Table 1: |||u - u_h|||_1, |||p_F|||_1, |||p_f|||_0, |||p_f|||_1, |||p_m|||_0,
    |||p_m|||_1 at the final time."""
    t = cfg["steps"] * cfg["dt"]
    Gp, Gc = M.region_grids(cfg, "h")
    F = ex1_functions(t)
    out = {}
    for k in ("pF", "pf", "pm"):
        l2, h1 = norms(Gp, np.ravel(fields[k]), *F[k])
        out[f"{k}_0"], out[f"{k}_1"] = l2, h1
    u = np.asarray(fields["u"]).reshape(2, -1)
    h1u2 = 0.0
    l2u2 = 0.0
    for a in range(2):
        l2, h1 = norms(Gc, u[a], *F[f"u{a}"])
        h1u2 += h1 * h1
        l2u2 += l2 * l2
    out["u_1"], out["u_0"] = np.sqrt(h1u2), np.sqrt(l2u2)
    return out
