"""Pins of the error-norm helper of the paper-protocol study (tests/protocol_norms.py): closed-form integrals
over the unit square (P:1465-1475 define the norms; the numbers below are plain calculus)."""
import numpy as np

import lpfem_inputs as I
from oracle import mesh as M
import protocol_norms as PN


def _grids(h):
    cfg = I.make_config(dim=2, H=2 * h, h=h, grid=1, dt=0.1, steps=1, problem="mms")
    Gp, Gc = M.region_grids(cfg, "h")
    box = M.Box(Gp, (0, 0), Gp.n)
    return Gp, Gp.coords(box.node_g)


def _fn(f, g):
    return (lambda P: f(P[:, 0], P[:, 1])), (lambda P: np.stack(g(P[:, 0], P[:, 1]), axis=1))


def test_norms_of_a_quadratic_are_exact():
    """||f||_0^2 = int (x^2+y^2)^2 = 28/45 and |f|_1^2 = int 4x^2+4y^2 = 8/3 on [0,1]^2 (u_h = 0)."""
    G, X = _grids(1 / 4)
    ex, gr = _fn(lambda x, y: x * x + y * y, lambda x, y: (2 * x, 2 * y))
    l2, h1 = PN.norms(G, np.zeros(X.shape[0]), ex, gr)
    assert abs(l2 * l2 - 28 / 45) < 1e-13 and abs(h1 * h1 - 8 / 3) < 1e-13


def test_interpolated_quadratic_has_zero_error():
    """P2 reproduces quadratics: I_h f - f = 0 (values, and gradients through grad lambda and d phi / d lambda)."""
    G, X = _grids(1 / 8)
    f = lambda x, y: 1 + x - 2 * y + 3 * x * x - x * y + 0.5 * y * y
    ex, gr = _fn(f, lambda x, y: (1 + 6 * x - y, -2 - x + y))
    l2, h1 = PN.norms(G, f(X[:, 0], X[:, 1]), ex, gr)
    assert l2 < 1e-13 and h1 < 1e-12


def test_seminorm_of_an_interpolated_linear_function():
    """u_h = I_h (2x + 3y), exact 0: |u_h|_1^2 = 13 |[0,1]^2| = 13, ||u_h||_0^2 = int (2x+3y)^2 = 4/3+3+3 = 22/3."""
    G, X = _grids(1 / 4)
    ex, gr = _fn(lambda x, y: 0 * x, lambda x, y: (0 * x, 0 * y))
    l2, h1 = PN.norms(G, 2 * X[:, 0] + 3 * X[:, 1], ex, gr)
    assert abs(h1 * h1 - 13) < 1e-12 and abs(l2 * l2 - 22 / 3) < 1e-12


def test_protocol_configs_follow_the_paper():
    """h = H^2, dt = h^2, T = 1, extension 1/4, 2x2 subdomains, all coefficients 1."""
    for lev, (H, h) in enumerate([(1 / 2, 1 / 4), (1 / 4, 1 / 16), (1 / 8, 1 / 64)]):
        c = PN.protocol_config(lev)
        assert c["H"] == H and c["h"] == h and c["dt"] == h * h and c["steps"] * c["dt"] == 1.0
        assert c["overlap"] == 0.25 and c["grid"] == [2, 2] and c["coeffs"]["k"] == [1.0, 1.0, 1.0]
