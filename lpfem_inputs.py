"""Seeded synthetic inputs shared by the CUDA path's harness and the oracle.

This module holds NO method arithmetic: only the five BASELINE.json configs as
plain dicts (geometry, mesh sizes, subdomain grid, coefficients, time step) and
the seeded log-normal permeability multipliers (reading C15).  It is
the only module imported by both ``oracle/`` and the product binding's callers.

Coefficient arrays are indexed 0 = matrix m, 1 = microfracture f, 2 = macrofracture F.
"""
from __future__ import annotations

import copy

import numpy as np

# C9: k_m = 1e-2, k_f = 1e-1, k_F = 1; phi = C = sigma = sigma* = alpha = mu = rho = eta = nu = 1
BASE_COEFFS = {
    "phi": [1.0, 1.0, 1.0],
    "C": [1.0, 1.0, 1.0],
    "k": [1e-2, 1e-1, 1.0],
    "sigma": 1.0,
    "sigma_star": 1.0,
    "mu_tilde": 1.0,
    "nu": 1.0,
    "rho": 1.0,
    "alpha": 1.0,
    "eta": 1.0,
}


def _geom(dim: int) -> dict:
    if dim == 2:
        return {"porous_lo": [0.0, 0.0], "porous_hi": [1.0, 1.0], "conduit_lo": [0.0, 1.0], "conduit_hi": [1.0, 2.0]}
    return {"porous_lo": [0.0, 0.0, 0.0], "porous_hi": [1.0, 1.0, 1.0],
            "conduit_lo": [0.0, 0.0, 1.0], "conduit_hi": [1.0, 1.0, 2.0]}


def make_config(dim: int, H: float, h: float, grid: int, dt: float, steps: int, problem: str,
                seed: int | None = None, name: str = "custom", **over) -> dict:
    cfg = {"name": name, "dim": dim, "H": H, "h": h, "overlap": H, "grid": [grid] * dim,
           "dt": dt, "steps": steps, "problem": problem, "coeffs": copy.deepcopy(BASE_COEFFS),
           "lag_mode": "composite", "pressure_constraint": "mean_zero", "inflow_peak": 1.0,
           "krylov_rtol": 1e-12, "seed": seed}
    cfg.update(_geom(dim))
    cfg.update(over)
    cfg["k_mult"] = None if seed is None else lognormal_k_mult(cfg, seed)
    return cfg


def n_coarse_cells(cfg: dict) -> int:
    n = 1
    for a in range(cfg["dim"]):
        n *= int(round((cfg["porous_hi"][a] - cfg["porous_lo"][a]) / cfg["H"]))
    return n


def lognormal_k_mult(cfg: dict, seed: int, sigma_log: float = 1.0) -> np.ndarray:
    """One multiplier exp(sigma_log Z), Z ~ N(0,1) i.i.d., per porous coarse cell, lexicographic x fastest (C15)."""
    z = np.random.default_rng(seed).standard_normal(n_coarse_cells(cfg))
    return np.exp(sigma_log * z)


CONFIGS = {
    0: dict(dim=2, H=1 / 4, h=1 / 16, grid=2, dt=0.1, steps=5, problem="mms", name="cfg0"),
    1: dict(dim=2, H=1 / 8, h=1 / 64, grid=4, dt=0.05, steps=10, problem="mms", name="cfg1"),
    2: dict(dim=2, H=1 / 16, h=1 / 256, grid=8, dt=0.01, steps=20, problem="injection", seed=2, name="cfg2"),
    3: dict(dim=3, H=1 / 4, h=1 / 16, grid=2, dt=0.1, steps=10, problem="mms", name="cfg3"),
    4: dict(dim=3, H=1 / 8, h=1 / 48, grid=4, dt=0.01, steps=20, problem="injection", seed=4, name="cfg4"),
}


def config(i: int, **over) -> dict:
    kw = dict(CONFIGS[i])
    kw.update(over)
    return make_config(**kw)


def fine_dofs(cfg: dict) -> int:
    """D = 3 (2N+1)^d + d (2N+1)^d + (N+1)^d summed over the region boxes."""
    d = cfg["dim"]
    tot = 0
    for lo, hi, reg in ((cfg["porous_lo"], cfg["porous_hi"], "p"), (cfg["conduit_lo"], cfg["conduit_hi"], "c")):
        n = [int(round((hi[a] - lo[a]) / cfg["h"])) for a in range(d)]
        p2 = int(np.prod([2 * k + 1 for k in n]))
        p1 = int(np.prod([k + 1 for k in n]))
        tot += 3 * p2 if reg == "p" else d * p2 + p1
    return tot
