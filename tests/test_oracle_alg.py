"""Pins of oracle/alg1.py and oracle/alg3.py: convergence orders, special cases, invariants.

* Algorithm 1 on a steady manufactured solution (Ex1/Ex2 frozen at
  t = 0, so backward Euler adds no time error): observed orders ~3 for the P2
  fields and ~2 for the P1 pressure (Theorem PTS-Results P:399-407 with r = 1
  and the nodal superconvergence-free max norm).  A dropped interface term or a
  wrong sign stalls the error at O(1).
* Algorithm 3 special cases that reduce to a textbook solver:
  H = h (corrections vanish, composite = Algorithm 1 on T_h); one subdomain per
  region (the porous composite is the fine Algorithm 1 porous step driven by the
  coarse flux; the conduit composite solves the Newton-linearised step exactly).
* Invariants: constant state preserved, zero data stays zero, modes A and B
  coincide on the first step (C2), every fine node written once (C3).
"""
import numpy as np
import pytest

import lpfem_inputs as I
from oracle import mesh as M
from oracle.alg1 import Alg1, saddle
from oracle.alg3 import Alg3


def _errs(a, t):
    p = a.prob
    st = a.state if hasattr(a, "state") else a.comp
    e = [np.abs(st[f] - p.porous(f, a.Xp, t)).max() for f in ("pF", "pf", "pm")]
    e.append(np.abs(st["u"] - p.velocity(a.Xc, t)).max())
    ep = st["p"] - p.pressure(a.Xc1, t)
    e.append(np.abs(ep).max())
    return np.array(e)


def _steady_alg1(dim, h, steps):
    cfg = I.config(0 if dim == 2 else 3, h=h, H=h, dt=1e3, problem="mms_steady")
    Gp, Gc = M.region_grids(cfg, "h")
    a = Alg1(cfg, Gp, Gc, 1)
    for _ in range(steps):
        a.step()
    return _errs(a, 0.0)


def test_alg1_convergence_orders_2d():
    e = [_steady_alg1(2, h, 40) for h in (1 / 4, 1 / 8, 1 / 16)]
    rate = np.log2(e[1] / e[2])
    assert (rate[:4] > 2.5).all(), rate  # P2 fields
    assert rate[4] > 1.8, rate  # P1 pressure
    assert e[2][3] < 2e-4 and e[2][4] < 3e-2


def test_alg1_convergence_orders_3d():
    e = [_steady_alg1(3, h, 25) for h in (1 / 2, 1 / 4)]
    rate = np.log2(e[0] / e[1])
    assert (rate[:4] > 1.8).all(), rate  # pre-asymptotic on these tiny meshes (order 3 asymptotically)
    assert rate[4] > 1.2, rate


def test_alg1_time_order_first_order():
    """Backward Euler: halving dt halves the error at fixed fine h (time error dominant)."""
    errs = []
    for dt in (0.1, 0.05):
        cfg = I.config(0, h=1 / 8, H=1 / 8, dt=dt)
        Gp, Gc = M.region_grids(cfg, "h")
        a = Alg1(cfg, Gp, Gc, 1)
        for _ in range(int(round(0.4 / dt))):
            a.step()
        errs.append(_errs(a, 0.4))
    r = errs[0][:4] / errs[1][:4]
    assert (r[[0, 1, 3]] > 1.6).all() and (r < 2.6).all() and r[2] > 1.3, r  # p_m: k_m = 1e-2, space error visible


def _small2d(**over):
    kw = dict(h=1 / 8, H=1 / 4, dt=0.1, steps=2)
    kw.update(over)
    return I.config(0, **kw)


def test_alg3_degenerate_H_equals_h():
    """H = h: the coarse step already solves the fine equations, so every correction vanishes (to Picard/LU
    round-off) and the composite equals Algorithm 1 on T_h."""
    cfg = _small2d(H=1 / 8)
    a = Alg3(cfg)
    for _ in range(2):
        a.step()
        for P in a.P:
            assert max(np.abs(P["e"][f]).max() for f in P["e"]) < 1e-10
        for C in a.C:
            assert np.abs(C["e"]).max() < 1e-10
        for f in ("pF", "pf", "pm", "u"):
            assert np.abs(a.comp[f] - a.coarse.state[f]).max() < 1e-10


def test_alg3_single_subdomain_porous_is_alg1_step_with_coarse_flux():
    """grid = 1: Omega_p1 = Omega_p, the correction form collapses to the fine Algorithm 1 porous step whose
    interface flux is the coarse u_cH^n and whose lagged partners are the composite (mode B)."""
    cfg = _small2d(grid=1)
    a = Alg3(cfg)
    before = a.fields()
    uH_n = a.coarse.state["u"].copy()
    a.step()
    # direct fine solve of eqs. fullypF..fullypm with coarse flux
    ref = Alg1(cfg, a.Gp, a.Gc, a.R)
    ref.state = {k: v.copy() for k, v in before.items()}
    # replace the fine conduit flux by the prolonged coarse flux
    from oracle.fem import prolongation
    gc = ref.box_c.node_g
    u_flux = np.stack([prolongation(a.GcH, gc, a.R, 2) @ uH_n[k] for k in range(2)])
    ref.state["u"] = u_flux
    ref.step()
    for f in ("pF", "pf", "pm"):
        assert np.abs(a.comp[f] - ref.state[f]).max() < 1e-11 * max(1, np.abs(ref.state[f]).max())


def test_alg3_single_subdomain_conduit_newton_residual():
    """grid = 1: the conduit composite (u, p) satisfies the Newton-linearised fine step about U = P u_cH^{n+1}
    (b_N(e,U)+b_N(U,e)+b_N(U,U) = b_N(u,U)+b_N(U,u)-b_N(U,U)) in full-field form."""
    cfg = _small2d(grid=1)
    a = Alg3(cfg)
    before = a.fields()
    a.step()
    C = a.C[0]
    ops, d = C["ops"], 2
    from oracle.fem import prolongation
    U = np.stack([C["Pr2"] @ a.coarse.state["u"][k] for k in range(d)])
    u, p = a.comp["u"], a.comp["p"]
    A = ops.A_lin + ops.fem.convection(U, 1.0) + ops.fem.convection_reaction(U, 1.0)
    t = 0.1
    old_pF = None
    # residual of momentum rows at free nodes
    Uf = U.ravel()
    res_v = A @ u.ravel() - ops.Bdiv.T @ p - ops.fem.convection(U, 1.0) @ Uf
    pFH0 = Alg3(cfg).coarse.state["pF"]  # coarse p_FH^0
    gam = C["gam"]
    pFg = np.zeros(u.shape[1])
    pFg[gam] = C["PpF"] @ pFH0
    rhs_v = ops.fem.vec_mass(1.0) @ a.prob.f(C["X"], t).ravel() + ops.Mu @ before["u"].ravel() + ops.gamma_load(pFg)
    free = np.concatenate([C["cls"] <= M.GAMMA] * d)
    r = (res_v - rhs_v)[free]
    assert np.abs(r).max() < 1e-10 * np.abs(rhs_v).max()
    assert np.abs(ops.Bdiv @ u.ravel()).max() < 1e-11


def test_alg3_constant_state_invariant():
    cfg = _small2d(problem="constant", const_value=2.5)
    a = Alg3(cfg)
    for _ in range(2):
        a.step()
    for f in ("pF", "pf", "pm"):
        assert np.abs(a.comp[f] - 2.5).max() < 1e-12
    assert np.abs(a.comp["u"]).max() < 1e-12
    assert np.abs(a.comp["p"] - 2.5).max() < 1e-11


def test_alg3_zero_data_stays_zero():
    cfg = _small2d(problem="injection", inflow_peak=0.0)
    a = Alg3(cfg)
    a.step()
    for k, v in a.comp.items():
        assert np.abs(v).max() == 0.0


def test_alg3_modes_coincide_first_step():
    ca = _small2d(lag_mode="subdomain")
    cb = _small2d(lag_mode="composite")
    a, b = Alg3(ca), Alg3(cb)
    a.step()
    b.step()
    for k in a.comp:
        assert np.abs(a.comp[k] - b.comp[k]).max() < 1e-12
    a.step()
    b.step()
    assert max(np.abs(a.comp[k] - b.comp[k]).max() for k in a.comp) > 1e-8  # they differ afterwards


def test_alg3_accuracy_close_to_alg1():
    """Soft trend (Theorem TheoremFinal; Tables 1-2): the local parallel composite error is of the
    same size as Algorithm 1 on T_h."""
    cfg = _small2d(steps=3)
    a = Alg3(cfg)
    ref = Alg1(cfg, a.Gp, a.Gc, a.R)
    for _ in range(3):
        a.step()
        ref.step()
    ea, er = _errs(a, 0.3), _errs(ref, 0.3)
    assert (ea[:4] < 3.0 * er[:4] + 1e-3).all(), (ea, er)
