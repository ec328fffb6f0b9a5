"""Problem data: manufactured solutions (SymPy) and the injection problem (oracle; test infrastructure).

* Ex1 (2D) exact solution.  Forcing, Dirichlet and initial data
  "derived from the analytical solutions".
* Ex2 (3D) exact solution, reflected into the BASELINE geometry
  (porous [0,1]^3 below the conduit [0,1]^2 x [1,2], Gamma z = 1) by
  z_paper = 1 - z, u_z -> -u_z, pressures unchanged (C17).
* Injection (cfg2/cfg4): zero forcing, zero initial state, unit parabolic inflow
  on the top conduit face, no-slip sides, p_i = 0 on dOmega_p \\ Gamma (C16).

Forcing from the strong form:
  q_F = phi_F C_F dp_F/dt - div(k_F/mu grad p_F) + sigma* k_f/mu (p_F - p_f)          (eq. 1)
  q_f = phi_f C_f dp_f/dt - div(k_f/mu grad p_f) + sigma* k_f/mu (p_f - p_F)
        + sigma k_m/mu (p_f - p_m)                                                   (eq. 2)
  q_m = phi_m C_m dp_m/dt - div(k_m/mu grad p_m) + sigma k_m/mu (p_m - p_f)           (eq. 3)
  f_c = du/dt - div(2 nu D(u) - p I) + (u . grad) u                                   (eq. 4)
computed symbolically by SymPy differentiation, then lambdified to NumPy.
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np
import sympy as S

FIELDS = ("pF", "pf", "pm")


def _ex1_symbols():
    x, y, t = S.symbols("x y t", real=True)
    pi = S.pi
    a = 2 - pi * S.sin(pi * x)
    sol = {
        "pm": a * S.sin(S.Rational(1, 2) * pi * (3 * y**3 - 2 * y**2)) * S.cos(t),
        "pf": a * S.cos(pi * (1 - y)) * S.cos(t),
        "pF": a * (1 - y - S.cos(pi * y)) * S.cos(t),
        "u": [(x**2 * (y - 1) ** 2 + y) * S.cos(t),
              -S.Rational(2, 3) * x * (y - 1) ** 3 * S.cos(t) + a * S.cos(t)],
        "p": a * S.sin(S.Rational(1, 2) * pi * y) * S.cos(t),
    }
    return (x, y), t, sol


def _ex2_reflected_symbols():
    x, y, z, t = S.symbols("x y z t", real=True)
    zp = 1 - z  # paper's z: Gamma at z_paper = 0, conduit z_paper <= 0
    e = S.exp(-t)
    sxy, cxy = S.sin(x * y), S.cos(x * y)
    r2 = x**2 + y**2
    pm = -zp + S.exp(zp) - e * sxy * S.cos(zp)
    pF = -zp + (-(x**2) - y**2 + 8) * e * sxy * S.cos(zp)
    ux = (2 * x * sxy + y * (r2 - 8) * cxy) * e
    uy = (2 * y * sxy + x * (r2 - 8) * cxy) * e
    uz_paper = 1 + (r2 * (r2 - 8) * sxy - 4 * sxy - 8 * x * y * cxy) * zp * e
    p = (-16 * x * y * cxy + (r2 + zp**2 - 8) * (2 * r2 + 2 * zp**2 - 1) * sxy - 8 * sxy) * e
    sol = {"pm": pm, "pf": pm, "pF": pF, "u": [ux, uy, -uz_paper], "p": p}
    return (x, y, z), t, sol


def _div(vec, X):
    return sum(S.diff(vec[a], X[a]) for a in range(len(X)))


def _lap(f, X):
    return sum(S.diff(f, xa, 2) for xa in X)


def forcing_symbols(sol, X, t, co):
    """Strong-form residuals of eqs. (1)-(4) for the symbolic solution sol."""
    mu = co["mu_tilde"]
    kF, kf, km = co["k"][2], co["k"][1], co["k"][0]
    phiC = [co["phi"][i] * co["C"][i] for i in range(3)]  # index 0 = m, 1 = f, 2 = F
    sFf = co["sigma_star"] * kf / mu
    sfm = co["sigma"] * km / mu
    pF, pf, pm = sol["pF"], sol["pf"], sol["pm"]
    q = {
        "pF": phiC[2] * S.diff(pF, t) - kF / mu * _lap(pF, X) + sFf * (pF - pf),
        "pf": phiC[1] * S.diff(pf, t) - kf / mu * _lap(pf, X) + sFf * (pf - pF) + sfm * (pf - pm),
        "pm": phiC[0] * S.diff(pm, t) - km / mu * _lap(pm, X) + sfm * (pm - pf),
    }
    u, p, nu = sol["u"], sol["p"], co["nu"]
    d = len(X)
    f = []
    for a in range(d):
        # div(T)_a = sum_b d_b (2 nu D_ab - p delta_ab)
        divT = sum(S.diff(nu * (S.diff(u[a], X[b]) + S.diff(u[b], X[a])) - (p if a == b else 0), X[b]) for b in range(d))
        conv = sum(u[b] * S.diff(u[a], X[b]) for b in range(d))
        f.append(S.diff(u[a], t) - divT + conv)
    return q, f


def _coeff_key(co):
    return tuple((k, tuple(v) if isinstance(v, (list, tuple)) else v) for k, v in sorted(co.items()) if k != "k_mult")


@lru_cache(maxsize=None)
def _mms_funcs(dim: int, ckey, steady: bool = False):
    co = dict(ckey)
    X, t, sol = _ex1_symbols() if dim == 2 else _ex2_reflected_symbols()
    if steady:  # the same fields frozen at t = 0 (convergence pins: no time-discretisation error)
        sol = {k: ([c.subs(t, 0) for c in v] if isinstance(v, list) else v.subs(t, 0)) for k, v in sol.items()}
    q, f = forcing_symbols(sol, X, t, co)
    args = list(X) + [t]
    lam = lambda e: S.lambdify(args, e, "numpy")
    out = {"exact": {k: lam(sol[k]) for k in ("pF", "pf", "pm", "p")},
           "u": [lam(c) for c in sol["u"]],
           "q": {k: lam(q[k]) for k in FIELDS},
           "f": [lam(c) for c in f]}
    return out


def _call(fn, X, t):
    v = fn(*[X[..., a] for a in range(X.shape[-1])], t)
    return np.broadcast_to(np.asarray(v, dtype=np.float64), X.shape[:-1]).copy()


class Problem:
    """Data of one configuration: exact/initial values, Dirichlet data and forcing at points."""

    def __init__(self, cfg: dict):
        self.kind = cfg["problem"]
        self.d = cfg["dim"]
        self.co = cfg["coeffs"]
        self.peak = cfg.get("inflow_peak", 1.0)
        self.const = cfg.get("const_value", 1.0)
        if self.kind in ("mms", "mms_steady"):
            self.F = _mms_funcs(self.d, _coeff_key(self.co), self.kind == "mms_steady")
            self.kind = "mms"
        elif self.kind == "constant":
            # p_F = p_f = p_m = c, u = 0, p = c / rho, zero forcing: an exact discrete steady state (invariant pin)
            pass
        elif self.kind != "injection":
            raise ValueError(self.kind)

    # porous pressures ------------------------------------------------------
    def porous(self, field: str, X: np.ndarray, t: float) -> np.ndarray:
        """Exact (MMS) / initial-and-boundary (injection: 0) value of p_F, p_f, p_m."""
        if self.kind == "mms":
            return _call(self.F["exact"][field], X, t)
        if self.kind == "constant":
            return np.full(X.shape[:-1], self.const)
        return np.zeros(X.shape[:-1])

    def q(self, field: str, X: np.ndarray, t: float) -> np.ndarray:
        if self.kind == "mms":
            return _call(self.F["q"][field], X, t)
        return np.zeros(X.shape[:-1])

    # conduit ---------------------------------------------------------------
    def velocity(self, X: np.ndarray, t: float, on_top=None) -> np.ndarray:
        """(d, N) exact velocity (MMS) or Dirichlet velocity (injection: inflow on the top face, C16)."""
        if self.kind == "mms":
            return np.stack([_call(c, X, t) for c in self.F["u"]])
        out = np.zeros((self.d,) + X.shape[:-1])
        if on_top is not None and self.kind == "injection":
            prof = np.ones(X.shape[:-1])
            for a in range(self.d - 1):
                prof = prof * 4.0 * X[..., a] * (1.0 - X[..., a])
            out[self.d - 1] = np.where(on_top, -self.peak * prof, 0.0)
        return out

    def pressure(self, X: np.ndarray, t: float) -> np.ndarray:
        if self.kind == "mms":
            return _call(self.F["exact"]["p"], X, t)
        if self.kind == "constant":
            return np.full(X.shape[:-1], self.const / self.co["rho"])
        return np.zeros(X.shape[:-1])

    def f(self, X: np.ndarray, t: float) -> np.ndarray:
        if self.kind == "mms":
            return np.stack([_call(c, X, t) for c in self.F["f"]])
        return np.zeros((self.d,) + X.shape[:-1])
