"""Pins of the oracle parts that round 1 left without one ("What's weak" 1).

* C15 (log-normal permeability, BASELINE configs 2/4): the multiplier of porous coarse cell c scales k_m, k_f,
  k_F on exactly the fine elements inside c (``alg1.coarse_cell_mult``), and the BJ friction / tangential Gamma
  terms of the conduit on exactly the Gamma facets above the porous coarse cell under them
  (``alg1._facet_mult_for``).  Pinned by a one-hot multiplier: the operator difference must equal a
  multiple of the operator assembled by ``BoxFEM`` on a box that covers only that coarse cell (or only the
  facets above it), embedded by half-grid index.  A transposed, offset or wrong-layer cell index fails.
* C16 (injection data): the inflow profile is the unit parabola 4x(1-x) (2D) / 16x(1-x)y(1-y) (3D) pointing
  into the conduit on the top face and zero on the side walls (closed-form point values), and the
  discrete Gamma flux of every coarse step equals the discrete inflow flux (2D: 2/3 exactly; 3D: the P2
  interpolant of the biquadratic profile, -> 4/9): summing the continuity rows (sum_k psi_k = 1) gives
  int div u_h = 0.
* C4 (pressure Q_0^h): ``Box.on_artificial`` against the face-centre test in physical coordinates.
* P2 prolongation weights reproduce every quadratic exactly (nesting).
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp

import lpfem_inputs as I
from oracle import mesh as M
from oracle.alg1 import Alg1, PorousOps, make_conduit_ops
from oracle.fem import BoxFEM, exact_prolong_weights


def _embed(sub_box: M.Box, big_box: M.Box, A_sub: sp.spmatrix, ncomp: int = 1) -> sp.csr_matrix:
    """Embed a matrix assembled on sub_box (P2 local numbering, ncomp component blocks) into big_box."""
    g = sub_box.node_g
    idx = big_box.p2_index(g)
    n_s, n_b = len(g), big_box.node_g.shape[0]
    full = np.concatenate([idx + c * n_b for c in range(ncomp)])
    A = sp.coo_matrix(A_sub)
    return sp.coo_matrix((A.data, (full[A.row], full[A.col])), shape=(ncomp * n_b, ncomp * n_b)).tocsr()


def _one_hot(cfg, cell, factor=10.0):
    nH = [int(round((cfg["porous_hi"][a] - cfg["porous_lo"][a]) / cfg["H"])) for a in range(cfg["dim"])]
    k = np.ones(int(np.prod(nH)))
    k[int(M.lex_index(np.asarray(cell), np.zeros(cfg["dim"], np.int64), np.asarray(nH)))] = factor
    return k


@pytest.mark.parametrize("dim,cell", [(2, (2, 1)), (2, (1, 2)), (3, (1, 0, 1))])
def test_c15_porous_multiplier_on_exactly_one_coarse_cell(dim, cell):
    """One-hot k_mult (cell c x 10): A_i(one-hot) - A_i(1) = 9 (k_i K_c + exchange M_c) with K_c, M_c assembled
    on the fine elements of coarse cell c alone (BASELINE cfg2/cfg4 'scaled per coarse cell', C15)."""
    base = I.config(0 if dim == 2 else 3, H=1 / 4, h=1 / 8 if dim == 2 else 1 / 8)
    R = 2
    Gp, _ = M.region_grids(base, "h")
    # a porous subdomain box that contains the coarse cell and more (cells [0, n) = whole region here)
    big = M.Box(Gp, (0,) * dim, Gp.n)
    ones = PorousOps(dict(base, k_mult=np.ones(len(_one_hot(base, cell)))), big, R)
    hot = PorousOps(dict(base, k_mult=_one_hot(base, cell)), big, R)
    c0 = tuple(R * c for c in cell)
    c1 = tuple(R * (c + 1) for c in cell)
    small = BoxFEM(M.Box(Gp, c0, c1))
    co = base["coeffs"]
    mu = co["mu_tilde"]
    k = co["k"]
    Kc = _embed(small.box, big, small.stiffness())
    Mc = _embed(small.box, big, small.mass())
    exp = {
        "pF": 9.0 * (k[2] / mu * Kc + co["sigma_star"] * k[1] / mu * Mc),
        "pf": 9.0 * (k[1] / mu * Kc + (co["sigma"] * k[0] + co["sigma_star"] * k[1]) / mu * Mc),
        "pm": 9.0 * (k[0] / mu * Kc + co["sigma"] * k[0] / mu * Mc),
    }
    for f in ("pF", "pf", "pm"):
        diff = (hot.A[f] - ones.A[f]) - exp[f]
        scale = np.abs(exp[f]).max()
        assert scale > 0
        assert np.abs(diff).max() <= 1e-12 * scale, f


def _conduit_facet_reference(cfg, Gc, big, tcell, R):
    """Friction facet mass and tangential-gradient matrices on the Gamma facets above porous coarse cell
    (tcell, top layer), embedded into the conduit box `big`."""
    d = cfg["dim"]
    c0 = tuple(R * c for c in tcell) + (0,)
    c1 = tuple(R * (c + 1) for c in tcell) + (1,)
    small = BoxFEM(M.Box(Gc, c0, c1))
    Mf = small.facet_mass(None)
    Tg = [small.facet_tangential_grad(a, None) for a in range(d - 1)]
    return small, Mf, Tg


@pytest.mark.parametrize("dim,tcell", [(2, (2,)), (3, (1, 2))])
def test_c15_gamma_friction_uses_the_porous_cell_under_the_facet(dim, tcell):
    """One-hot k_mult on the top-layer porous coarse cell under Gamma: the BJ friction eta nu alpha / sqrt(k_F)
     scales by 1/sqrt(10) and the tangential load coefficient eta nu alpha sqrt(k_F)/mu
    by sqrt(10) on exactly the facets above that cell; a one-hot cell NOT under Gamma changes nothing."""
    base = I.config(0 if dim == 2 else 3, H=1 / 4, h=1 / 8)
    R = 2
    _, Gc = M.region_grids(base, "h")
    big = M.Box(Gc, (0,) * dim, Gc.n)
    nH = int(round(1 / base["H"]))
    ones = make_conduit_ops(dict(base, k_mult=np.ones(nH ** dim)), big, R)
    top_cell = tuple(tcell) + (nH - 1,)
    hot = make_conduit_ops(dict(base, k_mult=_one_hot(base, top_cell)), big, R)
    co = base["coeffs"]
    kF = co["k"][2]
    fr = co["eta"] * co["nu"] * co["alpha"] / np.sqrt(kF)
    ct = co["eta"] * co["nu"] * co["alpha"] * np.sqrt(kF) / co["mu_tilde"]
    small, Mf, Tg = _conduit_facet_reference(base, Gc, big, tcell, R)
    n2 = big.node_g.shape[0]
    blocks = [Mf if a < dim - 1 else sp.csr_matrix(Mf.shape) for a in range(dim)]
    exp_fr = _embed(small.box, big, sp.block_diag(blocks), ncomp=dim) * (fr * (1 / np.sqrt(10.0) - 1.0))
    d_fr = (hot.Fr - ones.Fr) - exp_fr
    assert np.abs(exp_fr).max() > 0
    assert np.abs(d_fr).max() <= 1e-12 * np.abs(exp_fr).max()
    for a in range(dim - 1):
        exp_t = _embed(small.box, big, Tg[a]) * (ct * (np.sqrt(10.0) - 1.0))
        d_t = (hot.TG[a] - ones.TG[a]) - exp_t
        assert np.abs(exp_t).max() > 0
        assert np.abs(d_t).max() <= 1e-12 * np.abs(exp_t).max()
    # a hot cell one layer below Gamma leaves the conduit operators unchanged
    low = tuple(tcell) + (nH - 2,)
    other = make_conduit_ops(dict(base, k_mult=_one_hot(base, low)), big, R)
    assert np.abs(other.Fr - ones.Fr).max() == 0.0
    for a in range(dim - 1):
        assert np.abs(other.TG[a] - ones.TG[a]).max() == 0.0


def test_c15_lognormal_recipe():
    """C15: one exp(Z), Z ~ N(0,1) (numpy default_rng(seed)), per porous coarse cell: 256 (cfg2), 512 (cfg4),
    median-preserving (log-mean ~ 0, log-sd ~ 1)."""
    for i, n in ((2, 256), (4, 512)):
        cfg = I.config(i)
        k = np.asarray(cfg["k_mult"])
        assert k.shape == (n,)
        z = np.random.default_rng(i).standard_normal(n)
        assert np.array_equal(k, np.exp(z))
        assert abs(z.mean()) < 0.15 and 0.85 < z.std() < 1.15


@pytest.mark.parametrize("dim", [2, 3])
def test_c16_inflow_profile_point_values(dim):
    """Unit parabolic inflow directed into the conduit on its top face (C16): 2D u = (0, -4x(1-x)), 3D
    u = (0, 0, -16x(1-x)y(1-y)); zero on the side walls and in the tangential components."""
    from oracle.mms import Problem
    cfg = I.config(2 if dim == 2 else 4, h=1 / 4, H=1 / 2)
    pr = Problem(cfg)
    if dim == 2:
        X = np.array([[0.5, 2.0], [0.25, 2.0], [0.0, 2.0], [1.0, 2.0], [0.0, 1.5], [0.5, 1.5]])
        exp_last = np.array([-1.0, -0.75, 0.0, 0.0, 0.0, 0.0])
    else:
        X = np.array([[0.5, 0.5, 2.0], [0.25, 0.5, 2.0], [0.25, 0.75, 2.0], [0.0, 0.5, 2.0], [0.5, 1.0, 2.0],
                      [0.5, 0.5, 1.5]])
        exp_last = np.array([-1.0, -0.75, -0.5625, 0.0, 0.0, 0.0])
    on_top = X[:, -1] == 2.0
    on_top[-1] = False
    u = pr.velocity(X, 0.37, on_top)
    assert np.array_equal(u[-1], exp_last)
    assert np.all(u[:-1] == 0.0)
    u2 = Problem(dict(cfg, inflow_peak=2.5)).velocity(X, 0.37, on_top)
    assert np.array_equal(u2[-1], 2.5 * exp_last)


@pytest.mark.parametrize("dim,h", [(2, 1 / 8), (3, 1 / 4)])
def test_c16_gamma_flux_equals_inflow_flux(dim, h):
    """Every (coarse) step: int_Gamma u_h . e_last = int_top u_D . e_last = -2/3 (2D) / -4/9 (3D) at peak 1, to
    solver round-off.  The continuity rows sum to int div u_h = 0 (sum_k psi_k = 1 on the whole-region P1 space,
    Gamma natural), the side walls are no-slip, and the P2 interpolant of the quadratic inflow is exact.  Also
    the porous interface load int_Gamma (u.n_c) v_F sums to +2/3 / +4/9."""
    cfg = I.config(2 if dim == 2 else 4, h=h, H=h, dt=0.05, seed=None)
    Gp, Gc = M.region_grids(cfg, "h")
    a = Alg1(cfg, Gp, Gc, 1)
    MG = a.con.fem.facet_mass(None)
    if dim == 2:
        exact = -2.0 / 3.0  # 4x(1-x) is quadratic: its P2 interpolant is exact
    else:
        # 16x(1-x)y(1-y) is biquadratic (degree 4): the inflow is its P2 interpolant, whose face integral is
        # sum_i g(x_i) int phi_i; the top face carries the same tangential mesh as Gamma, so int phi_i is read
        # off the Gamma facet mass (1^T MG); -> 4/9 as h -> 0
        w = np.ones(MG.shape[0]) @ MG
        X = a.Xc
        g = 16 * X[:, 0] * (1 - X[:, 0]) * X[:, 1] * (1 - X[:, 1])
        exact = -float(w @ g)
        assert abs(exact + 4.0 / 9.0) < 1e-3
    for n in range(3):
        a.step()
        flux = np.ones(MG.shape[0]) @ (MG @ a.state["u"][-1])
        assert abs(flux - exact) <= 1e-12, (n, flux)
        assert abs(a.flux_load(a.state["u"]).sum() + exact) <= 1e-12
    assert np.abs(a.state["pF"]).max() > 0  # the interface flux drives the porous pressure


def test_c4_on_artificial_matches_face_centre_test():
    """Q_0^h of P:226 (reading C4): a box point is on the closure of the artificial faces iff it lies on a closed
    face of the box whose centre is interior to the region (physical coordinates)."""
    for cfgi in (0, 3):
        cfg = I.config(cfgi, h=1 / 8, H=1 / 4)
        d = cfg["dim"]
        for G in M.region_grids(cfg, "h"):
            ov = 2
            for sub in M.subdomains(G, tuple(cfg["grid"]), ov):
                box = sub.box
                g = box.node_g
                got = box.on_artificial(g)
                lo, hi = np.asarray(G.lo), np.asarray(G.hi)
                exp = np.zeros(len(g), bool)
                for a in range(d):
                    for side, c in ((0, box.c0[a]), (1, box.c1[a])):
                        centre = np.array([(box.c0[b] + box.c1[b]) / 2 for b in range(d)], float)
                        centre[a] = c
                        X = G.coords(2 * centre[None, :])[0]  # physical face centre
                        interior = np.all((X > lo + 1e-12) & (X < hi - 1e-12))
                        if interior:
                            exp |= g[:, a] == 2 * c
                assert np.array_equal(got, exp)


def test_prolongation_weights_reproduce_quadratics():
    """Exact rational P2 weights of a fine node reproduce every quadratic of the coarse cell (the nested P2 space
    contains the coarse one): sum_i w_i q(x_i) = q(x) for all monomials of degree <= 2."""
    for d, R in ((2, 4), (3, 3)):
        # coarse P2 nodes of the unit reference cell in the oracle's local order (vertices of the Kuhn simplex
        # containing the point, then edge midpoints) depend on the simplex: rebuild them the same way
        for num in itertools.product(range(2 * R + 1), repeat=d):
            xi = [Fraction(v, 2 * R) for v in num]
            order = sorted(range(d), key=lambda a: -xi[a])
            verts = [[Fraction(0)] * d]
            for k in range(d):
                v = list(verts[-1])
                v[order[k]] += 1
                verts.append(v)
            nodes = verts + [[(verts[a][c] + verts[b][c]) / 2 for c in range(d)]
                             for a, b in itertools.combinations(range(d + 1), 2)]
            w = exact_prolong_weights(d, num, R)
            assert len(w) == len(nodes)
            for pw in itertools.product(range(3), repeat=d):
                if sum(pw) > 2:
                    continue
                q = lambda x: np.prod([x[c] ** pw[c] for c in range(d)])
                assert sum(wi * q(xn) for wi, xn in zip(w, nodes)) == q(xi), (d, num, pw)
