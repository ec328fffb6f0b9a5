"""Pins of oracle/fem.py and oracle/mms.py against closed-form integrals, invariants and the PDE.

Each test evaluates an assembled form on fields whose integral is known in closed
form (textbook calculus on the unit square / cube), so a dropped term, a wrong
sign or a transposed operand in the oracle's assembly fails here.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla
import sympy as S

import lpfem_inputs as I
from oracle import mesh as M
from oracle.alg1 import make_conduit_ops, saddle
from oracle.alg3 import DirichletLU
from oracle.fem import BoxFEM, prolongation
from oracle import mms


def unit_box(d, n, region="p"):
    lo = (0.0,) * d if region == "p" else (0.0,) * (d - 1) + (1.0,)
    hi = (1.0,) * d if region == "p" else (1.0,) * (d - 1) + (2.0,)
    g = M.Grid(region, lo, hi, (n,) * d)
    return g, M.Box(g, (0,) * d, g.n)


@pytest.mark.parametrize("d,n", [(2, 3), (3, 2)])
def test_mass_stiffness_closed_forms(d, n):
    g, box = unit_box(d, n)
    fem = BoxFEM(box)
    X = g.coords(box.node_g)
    Mm, K = fem.mass(), fem.stiffness()
    one = np.ones(len(X))
    assert abs(one @ Mm @ one - 1.0) < 1e-13  # |Omega|
    assert abs(one @ Mm @ X[:, 0] - 0.5) < 1e-13  # int x
    assert abs(X[:, 0] @ Mm @ X[:, 0] - 1 / 3) < 1e-13  # int x^2
    assert abs(K - K.T).max() < 1e-13
    assert np.abs(K @ one).max() < 1e-12  # constants in the kernel
    # int |grad u|^2 for u = x^2 + x y (P2-exact): grad = (2x + y, x) -> int (2x+y)^2 + x^2 = 4/3 + 1 + 1/3 + 1/3
    u = X[:, 0] ** 2 + X[:, 0] * X[:, 1]
    assert abs(u @ K @ u - (4 / 3 + 1.0 + 1 / 3 + 1 / 3)) < 1e-12


@pytest.mark.parametrize("d,n", [(2, 3), (3, 2)])
def test_deformation_divergence_convection(d, n):
    g, box = unit_box(d, n, "c")
    fem = BoxFEM(box)
    X = g.coords(box.node_g)
    N = len(X)
    A = fem.deformation(1.0)  # 2 (D u, D v)
    # rigid motions: translations and the rotation (-y, x) in the kernel
    for a in range(d):
        t = np.zeros((d, N))
        t[a] = 1.0
        assert np.abs(A @ t.ravel()).max() < 1e-12
    rot = np.zeros((d, N))
    rot[0], rot[1] = -X[:, 1], X[:, 0]
    assert np.abs(A @ rot.ravel()).max() < 1e-12
    # u = (y^2, 0, ..): D = [[0, y],[y, 0]], 2 int D:D = 2 int 2 y^2 = 4 int y^2
    # (y in [1,2] in 2D: int y^2 = 7/3; y in [0,1] in 3D: 1/3)
    iy, iy2 = (1.5, 7 / 3) if d == 2 else (0.5, 1 / 3)
    u = np.zeros((d, N))
    u[0] = X[:, 1] ** 2
    assert abs(u.ravel() @ A @ u.ravel() - 4 * iy2) < 1e-11
    # divergence: B (y^2, x^2) = 0 (divergence-free quadratic); p = 1, u = (x, 0): eta int div u = eta
    B = fem.divergence(2.0)
    w = np.zeros((d, N))
    w[0], w[1] = X[:, 1] ** 2, X[:, 0] ** 2
    assert np.abs(B @ w.ravel()).max() < 1e-12
    u = np.zeros((d, N))
    u[0] = X[:, 0]
    assert abs(np.ones(B.shape[0]) @ B @ u.ravel() - 2.0) < 1e-12
    # convection eta ((w.grad) u, v): w = (x, 0), u = (x^2, 0), v = (1, 0): int x * 2x = 2/3
    wv = np.zeros((d, N))
    wv[0] = X[:, 0]
    Nw = fem.convection(wv, 1.0)
    u = np.zeros((d, N))
    u[0] = X[:, 0] ** 2
    v = np.zeros((d, N))
    v[0] = 1.0
    assert abs(v.ravel() @ Nw @ u.ravel() - 2 / 3) < 1e-12
    # reaction ((e.grad) U, v): e = (1, 0), U = (x^2 y, 0), v = (1, 0): int 2 x y = 2 * 1/2 * int y
    U = np.zeros((d, N))
    U[0] = X[:, 0] ** 2 * X[:, 1]
    Rt = fem.convection_reaction(U, 1.0)
    e = np.zeros((d, N))
    e[0] = 1.0
    assert abs(v.ravel() @ Rt @ e.ravel() - iy) < 1e-12
    # Newton pair consistency: N(U) U == R(U) U  (both are ((U.grad) U, v))
    U[1] = X[:, 0] * X[:, 1]
    assert np.abs(fem.convection(U, 1.0) @ U.ravel() - fem.convection_reaction(U, 1.0) @ U.ravel()).max() < 1e-12


@pytest.mark.parametrize("d,n", [(2, 3), (3, 2)])
def test_gamma_facet_forms(d, n):
    """Facet mass / tangential gradient on Gamma (bottom face of the conduit box)."""
    g, box = unit_box(d, n, "c")
    fem = BoxFEM(box)
    X = g.coords(box.node_g)
    MG = fem.facet_mass()
    one = np.ones(len(X))
    assert abs(one @ MG @ one - 1.0) < 1e-13  # |Gamma|
    assert abs(one @ MG @ X[:, 0] ** 2 - 1 / 3) < 1e-13
    T0 = fem.facet_tangential_grad(0)
    assert np.abs(T0 @ one).max() < 1e-13  # tangential gradient of a constant
    assert abs(one @ T0 @ X[:, 0] ** 2 - 1.0) < 1e-13  # int_Gamma 2x
    # nodes off Gamma carry nothing
    off = box.node_g[:, -1] != 0
    assert np.abs(MG[off]).max() == 0


@pytest.mark.parametrize("d,R", [(2, 4), (3, 2)])
def test_prolongation_exact_on_coarse_functions(d, R):
    """P evaluates coarse P2 / P1 functions exactly at fine nodes (nested meshes): reproduce quadratics / linears."""
    gH = M.Grid("p", (0.0,) * d, (1.0,) * d, (2,) * d)
    gh = M.Grid("p", (0.0,) * d, (1.0,) * d, (2 * R,) * d)
    bH, bh = M.Box(gH, (0,) * d, gH.n), M.Box(gh, (0,) * d, gh.n)
    rng = np.random.default_rng(0)
    c = rng.standard_normal((d + 1, d + 1))
    q = lambda X: c[0, 0] + X @ c[0, 1:] + sum(c[a + 1, b + 1] * X[:, a] * X[:, b] for a in range(d) for b in range(d))
    P2 = prolongation(gH, bh.node_g, R, 2)
    assert np.abs(P2 @ q(gH.coords(bH.node_g)) - q(gh.coords(bh.node_g))).max() < 1e-12
    lin = lambda X: c[0, 0] + X @ c[0, 1:]
    P1 = prolongation(gH, bh.vert_g, R, 1)
    assert np.abs(P1 @ lin(gH.coords(bH.vert_g)) - lin(gh.coords(bh.vert_g))).max() < 1e-12


def test_dense_bruteforce_vs_superlu():
    """The SuperLU subdomain solve equals a dense numpy solve on a tiny bordered saddle system."""
    cfg = I.config(0, h=1 / 4, H=1 / 4)
    g = M.Grid("c", (0.0, 1.0), (1.0, 2.0), (4, 4))
    box = M.Box(g, (1, 1), (4, 4))  # enclosed: does not touch Gamma (y = 1)
    ops = make_conduit_ops(cfg, box, 1)
    d, n2, n1 = 2, box.node_g.shape[0], box.vert_g.shape[0]
    rng = np.random.default_rng(1)
    U = rng.standard_normal((d, n2))
    A = saddle(ops.A_lin + ops.fem.convection(U, 1.0) + ops.fem.convection_reaction(U, 1.0), ops.Bdiv)
    cls = box.classes()
    fixed = np.concatenate([cls >= M.ART] * d + [np.zeros(n1, bool)])
    border = np.concatenate([np.zeros(d * n2), ops.fem.p1_mass_vector()])
    b = rng.standard_normal(A.shape[0])
    vals = rng.standard_normal(int(fixed.sum()))
    x = DirichletLU(A, fixed, border).solve(b, vals)
    free = ~fixed
    Ad = A.toarray()
    Aff = Ad[np.ix_(free, free)]
    m = border[free]
    K = np.block([[Aff, m[:, None]], [m[None, :], np.zeros((1, 1))]])
    r = np.concatenate([b[free] - Ad[np.ix_(free, fixed)] @ vals, [0.0]])
    xd = np.linalg.solve(K, r)
    assert np.abs(x[free] - xd[:-1]).max() / np.abs(xd).max() < 1e-12
    assert abs(m @ x[free]) < 1e-10  # mean-zero pressure (C6)


# --------------------------------------------------------------------------- MMS
def _interface_residuals(dim):
    co = I.BASE_COEFFS
    if dim == 2:
        X, t, sol = mms._ex1_symbols()
        gam = {X[1]: 1}
        nc = [0, -1]
    else:
        X, t, sol = mms._ex2_reflected_symbols()
        gam = {X[2]: 1}
        nc = [0, 0, -1]
    d = len(X)
    u, p = sol["u"], sol["p"]
    nu, kF, mu, rho, alpha = co["nu"], co["k"][2], co["mu_tilde"], co["rho"], co["alpha"]
    T = [[nu * (S.diff(u[a], X[b]) + S.diff(u[b], X[a])) - (p if a == b else 0) for b in range(d)] for a in range(d)]
    Tn = [sum(T[a][b] * nc[b] for b in range(d)) for a in range(d)]
    npor = [-v for v in nc]
    gradF = [S.diff(sol["pF"], xa) for xa in X]
    res = {
        "div": sum(S.diff(u[a], X[a]) for a in range(d)),
        "mass": sum(u[a] * nc[a] for a in range(d)) - kF / mu * sum(gradF[a] * npor[a] for a in range(d)),
        "normal": -sum(nc[a] * Tn[a] for a in range(d)) - sol["pF"] / rho,
        "noflux_f": sum(S.diff(sol["pf"], X[a]) * npor[a] for a in range(d)),
        "noflux_m": sum(S.diff(sol["pm"], X[a]) * npor[a] for a in range(d)),
    }
    fric = alpha * nu * S.sqrt(d) / S.sqrt(d * kF)  # alpha nu sqrt(d) / sqrt(tr Pi), Pi = k_F I
    for a in range(d - 1):  # tangential components of P_tau
        res[f"BJ{a}"] = -Tn[a] - fric * (u[a] + kF / mu * gradF[a])
    return X, t, res, gam


@pytest.mark.parametrize("dim", [2, 3])
def test_mms_satisfies_interface_conditions(dim):
    """The (reflected) manufactured solutions satisfy eqs. (5)-(9) on Gamma at the config coefficients."""
    X, t, res, gam = _interface_residuals(dim)
    rng = np.random.default_rng(3)
    for name, r in res.items():
        f = S.lambdify(list(X) + [t], r if name == "div" else r.subs(gam), "numpy")
        for _ in range(20):
            pt = rng.uniform(0, 1, len(X))
            if name == "div":
                pt[-1] += 1.0
            v = f(*pt, rng.uniform(0, 1))
            assert abs(v) < 1e-10, (name, v)


@pytest.mark.parametrize("dim", [2, 3])
def test_mms_forcing_finite_difference_residual(dim):
    """Lambdified forcing equals the PDE operator applied by central finite differences."""
    cfg = I.config(0 if dim == 2 else 3)
    pr = mms.Problem(cfg)
    co = cfg["coeffs"]
    rng = np.random.default_rng(5)
    hfd = 1e-3
    for _ in range(30):
        x = rng.uniform(0.1, 0.9, dim)
        xc = x.copy()
        xc[-1] += 1.0
        t = rng.uniform(0.1, 1.0)
        E = np.eye(dim) * hfd
        P = lambda f, y, s: pr.porous(f, y[None], s)[0]
        lap = lambda f, y, s: sum((P(f, y + E[a], s) - 2 * P(f, y, s) + P(f, y - E[a], s)) / hfd**2 for a in range(dim))
        dtf = lambda f, y, s: (P(f, y, s + hfd) - P(f, y, s - hfd)) / (2 * hfd)
        kF, kf, km = co["k"][2], co["k"][1], co["k"][0]
        qF = dtf("pF", x, t) - kF * lap("pF", x, t) + kf * (P("pF", x, t) - P("pf", x, t))
        qf = dtf("pf", x, t) - kf * lap("pf", x, t) + kf * (P("pf", x, t) - P("pF", x, t)) + km * (P("pf", x, t) - P("pm", x, t))
        qm = dtf("pm", x, t) - km * lap("pm", x, t) + km * (P("pm", x, t) - P("pf", x, t))
        for name, v in (("pF", qF), ("pf", qf), ("pm", qm)):
            assert abs(pr.q(name, x[None], t)[0] - v) < 1e-5 * max(1, abs(v))
        # momentum: du/dt - nu lap u - nu grad div u + grad p + (u.grad) u
        V = lambda y, s: pr.velocity(y[None], s)[:, 0]
        p = lambda y: pr.pressure(y[None], t)[0]
        u0 = V(xc, t)
        for a in range(dim):
            du = (V(xc, t + hfd)[a] - V(xc, t - hfd)[a]) / (2 * hfd)
            lapu = sum((V(xc + E[b], t)[a] - 2 * u0[a] + V(xc - E[b], t)[a]) / hfd**2 for b in range(dim))
            graddiv = 0.0
            for b in range(dim):  # d_a d_b u_b
                graddiv += (V(xc + E[a] + E[b], t)[b] - V(xc + E[a] - E[b], t)[b] - V(xc - E[a] + E[b], t)[b]
                            + V(xc - E[a] - E[b], t)[b]) / (4 * hfd**2)
            dp = (p(xc + E[a]) - p(xc - E[a])) / (2 * hfd)
            conv = sum(u0[b] * (V(xc + E[b], t)[a] - V(xc - E[b], t)[a]) / (2 * hfd) for b in range(dim))
            fa = du - co["nu"] * (lapu + graddiv) + dp + conv
            assert abs(pr.f(xc[None], t)[a, 0] - fa) < 1e-4 * max(1, abs(fa))
