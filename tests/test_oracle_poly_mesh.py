"""Pins of oracle/poly.py and oracle/mesh.py against closed forms and the paper's worked layout.

None of these re-derive the oracle's formula: they check it against textbook
element matrices, an independent numerical quadrature, integer geometry and the
paper's printed Ex1 subdomains (tests/golden/ex1_layout.txt).
"""
import itertools
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy.special import roots_legendre

import lpfem_inputs as I
from oracle import mesh as M
from oracle import poly
from oracle.fem import BoxFEM, exact_prolong_weights

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _duffy_integral(alpha, d, n=12):
    """int over the reference d-simplex of prod lambda^alpha by collapsed (Duffy) Gauss-Legendre; /|K|."""
    x, w = roots_legendre(n)
    x = 0.5 * (x + 1)
    w = 0.5 * w
    tot = 0.0
    for idx in itertools.product(range(n), repeat=d):
        # collapsed coordinates: y1 = u1, y2 = (1 - u1) u2, y3 = (1 - u1)(1 - u2) u3
        u = [x[i] for i in idx]
        wt = np.prod([w[i] for i in idx])
        y, scale = [], 1.0
        for k in range(d):
            y.append(scale * u[k])
            jac = scale
            scale *= 1 - u[k]
            wt *= jac
        lam = [1 - sum(y)] + y
        tot += wt * np.prod([lam[i] ** alpha[i] for i in range(d + 1)])
    vol = 1.0 / np.prod(range(1, d + 1))
    return tot / vol


@pytest.mark.parametrize("d", [1, 2, 3])
def test_monomial_integral_matches_quadrature(d):
    for alpha in [(0,) * (d + 1), (2,) + (0,) * d, (1, 1) + (0,) * (d - 1), (2, 1, 2) + (0,) * (d - 2) if d >= 2 else (3, 2),
                  tuple(range(d + 1))]:
        assert abs(float(poly.monomial_integral(alpha)) - _duffy_integral(alpha, d)) < 1e-13


def test_p2_triangle_mass_textbook():
    """P2 triangle mass matrix = |K|/180 [6 vv, -1 vv', -4 vertex/opposite edge, 0 vertex/adjacent edge, 32 ee, 16 ee']."""
    T = poly.tensors(2)["mass22"]
    eds = poly.edges(2)
    exp = np.zeros((6, 6), dtype=object)
    for i in range(6):
        for j in range(6):
            if i < 3 and j < 3:
                exp[i, j] = Fraction(6 if i == j else -1, 180)
            elif i >= 3 and j >= 3:
                exp[i, j] = Fraction(32 if i == j else 16, 180)
            else:
                v, e = (i, eds[j - 3]) if i < 3 else (j, eds[i - 3])
                exp[i, j] = Fraction(0 if v in e else -4, 180)
    # the oracle's tensor is int / |K|
    assert all(T[i, j] == exp[i, j] for i in range(6) for j in range(6))


@pytest.mark.parametrize("d", [2, 3])
def test_p2_basis_integrals_textbook(d):
    """int phi_vertex = 0 (triangle), -|K|/20 (tet); int phi_edge = |K|/3 (triangle), |K|/5 (tet)."""
    m = poly.tensors(d)["mass22"]
    row = [sum(m[i, j] for j in range(m.shape[1])) for i in range(m.shape[0])]  # sum_j int phi_i phi_j = int phi_i
    v_exp = Fraction(0) if d == 2 else Fraction(-1, 20)
    e_exp = Fraction(1, 3) if d == 2 else Fraction(1, 5)
    assert all(r == v_exp for r in row[: d + 1])
    assert all(r == e_exp for r in row[d + 1:])


@pytest.mark.parametrize("d", [2, 3])
def test_p1_mass_closed_form(d):
    m = poly.tensors(d)["mass11"]
    for i in range(d + 1):
        for j in range(d + 1):
            assert m[i, j] == Fraction(1 + (i == j), (d + 1) * (d + 2))


@pytest.mark.parametrize("d,n", [(2, (3, 4)), (3, (2, 3, 2))])
def test_mesh_counts_and_volume(d, n):
    g = M.Grid("p", (0.0,) * d, tuple(float(k) / 4 for k in n), n)
    box = M.Box(g, (0,) * d, n)
    assert box.node_g.shape[0] == np.prod([2 * k + 1 for k in n])
    assert box.vert_g.shape[0] == np.prod([k + 1 for k in n])
    p2, p1, gv, cell = box.simplices()
    assert p2.shape[0] == np.prod(range(1, d + 1)) * np.prod(n)
    fem = BoxFEM(box)
    assert abs(fem.vol.sum() - np.prod([k / 4 for k in n])) < 1e-14
    # every P2 node and P1 vertex is used
    assert len(np.unique(p2)) == box.node_g.shape[0]
    assert len(np.unique(p1)) == box.vert_g.shape[0]


@pytest.mark.parametrize("d,R", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_kuhn_meshes_nested(d, R):
    """Each fine simplex lies in exactly one coarse Kuhn simplex (integer ordering test, C22)."""
    nH = (2,) * d
    gf = M.Grid("p", (0.0,) * d, (1.0,) * d, tuple(k * R for k in nH))
    box = M.Box(gf, (0,) * d, gf.n)
    _, _, gv, _ = box.simplices()
    v = gv // 2  # fine vertex integer coords (E, d+1, d)
    cen = v.sum(axis=1)  # (d+1) * centroid
    cell = cen // ((d + 1) * R)
    loc = v - (cell * R)[:, None, :]  # local numerators over R
    assert loc.min() >= 0 and loc.max() <= R
    cloc = cen - (d + 1) * R * cell
    order = np.argsort(-cloc, axis=1, kind="stable")
    for k in range(d - 1):
        a = np.take_along_axis(loc, order[:, None, k:k + 1].repeat(d + 1, 1), 2)[..., 0]
        b = np.take_along_axis(loc, order[:, None, k + 1:k + 2].repeat(d + 1, 1), 2)[..., 0]
        assert (a >= b).all()


def test_cfg0_layout_equals_paper_ex1():
    """cfg0's 2x2 per region, overlap H = 1/4, equals the printed D_j / Omega_j of Ex1."""
    cfg = I.config(0)
    Gp, Gc = M.region_grids(cfg, "h")
    ov = int(round(cfg["overlap"] / cfg["h"]))
    got = set()
    for G in (Gp, Gc):
        for s in M.subdomains(G, tuple(cfg["grid"]), ov):
            h = cfg["h"]
            core = tuple((G.lo[a] + s.core0[a] * h, G.lo[a] + s.core1[a] * h) for a in range(2))
            ext = tuple((G.lo[a] + s.box.c0[a] * h, G.lo[a] + s.box.c1[a] * h) for a in range(2))
            got.add((G.region, core, ext))
    want = set()
    for line in open(os.path.join(GOLDEN, "ex1_layout.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        reg, *vals = line.split()
        f = [float(Fraction(v)) for v in vals]
        want.add((reg, ((f[0], f[1]), (f[2], f[3])), ((f[4], f[5]), (f[6], f[7]))))
    assert got == want


@pytest.mark.parametrize("cfgi", [0, 1, 3])
def test_ownership_partition(cfgi):
    """Every fine node is owned by exactly one subdomain, inside that subdomain's closed core (C3)."""
    cfg = I.config(cfgi)
    Gp, Gc = M.region_grids(cfg, "h")
    ov = int(round(cfg["overlap"] / cfg["h"]))
    m = tuple(cfg["grid"])
    for G in (Gp, Gc):
        allg = M.Box(G, (0,) * G.d, G.n).node_g
        own = M.owner(allg, G, m)
        subs = M.subdomains(G, m, ov)
        count = np.zeros(len(allg), int)
        for j, s in enumerate(subs):
            mine = own == j
            g = allg[mine]
            assert (g >= 2 * np.asarray(s.core0)).all() and (g <= 2 * np.asarray(s.core1)).all()
            count[mine] += 1
        assert (count == 1).all()


def test_node_class_precedence_2d():
    g = M.Grid("c", (0.0, 1.0), (1.0, 2.0), (8, 8))
    pts = np.array([[0, 0], [4, 0], [16, 8], [8, 8], [8, 4], [8, 16], [6, 6]])
    cls = g.classify(pts, (0, 0), (4, 4))  # box cells [0,4)^2: artificial faces at g = 8
    # (0,0): dir beats Gamma; (4,0): Gamma; (16,8): dir; (8,8): art corner; (8,4): art; (8,16): dir beats art; (6,6): int
    assert list(cls) == [M.DIR, M.GAMMA, M.DIR, M.ART, M.ART, M.DIR, M.INT]


def test_prolongation_weights_partition_of_unity():
    """Exact rational weights sum to one (constants reproduced); quadratic reproduction is pinned by
    tests/test_oracle_pins_r2.py::test_prolongation_weights_reproduce_quadratics."""
    for d, R in ((2, 4), (3, 3)):
        for num in itertools.product(range(2 * R + 1), repeat=d):
            w = exact_prolong_weights(d, num, R)
            assert sum(w) == 1
