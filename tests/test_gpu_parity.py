"""GPU parity: the CUDA path through the C-ABI against the independent CPU oracle (oracle/), on the
same seeded synthetic inputs.  Bar (BASELINE north_star, C20): relative l2 <= 1e-9 per field per step,
mesh and DOF indexing bit-exact (C21)."""
import numpy as np
import pytest

import lpfem_inputs as I
from gpu_helpers import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2311_05170_b200 import build
    build.build()


def run_pair(cfg, steps=None):
    from oracle import alg3
    from paper_2311_05170_b200 import LPFEM
    steps = cfg["steps"] if steps is None else steps
    ora = alg3.Alg3(cfg)
    sim = LPFEM(cfg)
    worst = {}
    for n in range(steps):
        ora.step()
        sim.step()
        errs, bad = compare(sim.fields(), ora.fields())
        for k, v in errs.items():
            worst[k] = max(worst.get(k, 0.0), v)
        assert not bad, f"step {n + 1}: {errs} stats={sim.stats()}"
    st = sim.stats()
    sim.close()
    return worst, st


def test_mesh_indexing_bit_exact_cfg0():
    from oracle import mesh as M
    from paper_2311_05170_b200 import LPFEM
    cfg = I.config(0)
    sim = LPFEM(cfg)
    for which, (lev, reg) in enumerate([("H", 0), ("H", 1), ("h", 0), ("h", 1)]):
        Gp, Gc = M.region_grids(cfg, lev)
        G = (Gp, Gc)[reg]
        box = M.Box(G, (0,) * cfg["dim"], G.n)
        coords, cells = sim.mesh(which)
        assert np.array_equal(coords, G.coords(box.node_g))
        p2, _, _, _ = box.simplices()
        assert np.array_equal(cells, p2)
    sim.close()


def test_layout_matches_oracle_cfg0():
    from oracle import mesh as M
    from paper_2311_05170_b200 import LPFEM
    cfg = I.config(0)
    sim = LPFEM(cfg)
    lay = sim.layout()
    Gp, Gc = M.region_grids(cfg, "h")
    subs = M.subdomains(Gp, tuple(cfg["grid"]), 4) + M.subdomains(Gc, tuple(cfg["grid"]), 4)
    assert len(lay) == len(subs)
    for L, S in zip(lay, subs):
        assert L["region"] == S.region
        assert L["core0"] == S.core0 and L["core1"] == S.core1
        assert L["box0"] == S.box.c0 and L["box1"] == S.box.c1
    sim.close()


def test_parity_cfg0_composite():
    worst, st = run_pair(I.config(0))
    print("cfg0 worst", worst, st)


def test_parity_cfg0_subdomain_lag():
    run_pair(I.config(0, lag_mode="subdomain"), steps=3)


def test_parity_constant_state_2d():
    cfg = I.config(0, problem="constant", steps=2)
    run_pair(cfg)


def test_parity_injection_lognormal_small_2d():
    # cfg2's structure (injection, log-normal k per coarse cell) on cfg0's mesh sizes
    cfg = I.make_config(dim=2, H=1 / 4, h=1 / 16, grid=2, dt=0.01, steps=4, problem="injection", seed=2)
    run_pair(cfg)


def test_parity_injection_lognormal_3d_full_trajectory():
    """cfg4's structure at a size the oracle marches in test time: 3D injection (C16: the biquadratic inflow on
    z = 2, no-slip sides) with the seeded log-normal permeability per porous coarse cell (C15, seed 4: the
    multiplier enters the porous operators and the BJ friction / tangential Gamma terms of the conduit boxes
    touching Gamma), 2x2x2 subdomains per region, both regions, every step to t_4 (the lag chain makes
    p_F, p_f, p_m non-zero from steps 2, 3, 4)."""
    cfg = I.make_config(dim=3, H=1 / 4, h=1 / 8, grid=2, dt=0.01, steps=4, problem="injection", seed=4)
    worst, st = run_pair(cfg)
    print("3d injection lognormal worst", worst)


def test_parity_3d_small_mms():
    cfg = I.make_config(dim=3, H=1 / 2, h=1 / 4, grid=2, dt=0.1, steps=2, problem="mms")
    run_pair(cfg)


def test_parity_cfg1_full_trajectory():
    worst, st = run_pair(I.config(1))
    print("cfg1 worst", worst)


# ---- edge cases: degenerate and ragged layouts (C5, C7, C8; SURVEY 8(c) c.3 "Coarse = fine degeneracy")

def test_parity_degenerate_H_equals_h():
    """H = h: the coarse step already solves the fine equations, every correction vanishes and the composite
    equals the coarse state (same mesh), on the GPU as in the oracle."""
    from paper_2311_05170_b200 import LPFEM
    cfg = I.make_config(dim=2, H=1 / 8, h=1 / 8, grid=2, dt=0.1, steps=2, problem="mms")
    run_pair(cfg)
    sim = LPFEM(cfg)
    for _ in range(2):
        sim.step()
    comp, coarse = sim.fields(), sim.coarse_fields()
    for f in ("pF", "pf", "pm", "u"):
        assert np.abs(np.ravel(comp[f]) - np.ravel(coarse[f])).max() < 1e-10, f
    sim.close()


def test_parity_single_subdomain_per_region():
    """One subdomain per region: the extended box is the whole region (overlap clipped at the boundary)."""
    run_pair(I.make_config(dim=2, H=1 / 4, h=1 / 16, grid=1, dt=0.1, steps=2, problem="mms"))


def test_parity_ragged_3x3_layout():
    """3 x 3 subdomains: corner, edge and interior boxes of three different shapes (C7 clipping)."""
    run_pair(I.make_config(dim=2, H=1 / 6, h=1 / 24, grid=3, dt=0.05, steps=2, problem="mms"))


def test_parity_3d_subdomain_lag():
    run_pair(I.make_config(dim=3, H=1 / 2, h=1 / 4, grid=2, dt=0.1, steps=2, problem="mms", lag_mode="subdomain"))


def test_misaligned_layout_fails_loudly():
    """Cores that do not fall on coarse grid lines are rejected (S:78 MisalignedLayout), not rounded."""
    from paper_2311_05170_b200 import LPFEM, LPFEMError
    cfg = I.make_config(dim=2, H=1 / 4, h=1 / 16, grid=3, dt=0.1, steps=1, problem="mms")
    with pytest.raises(LPFEMError):
        LPFEM(cfg)


def test_dt_change_reassembles_and_converges():
    """A different dt in lpfem_step re-assembles the dt-dependent operators and rebuilds the coarse-box inverses
    (header: porous matrices cached per dt); the warm-started Krylov solves still meet C19 and the state stays
    finite.  (The oracle marches with one dt, so this is a consistency check, not a parity check.)"""
    from paper_2311_05170_b200 import LPFEM
    cfg = I.make_config(dim=2, H=1 / 4, h=1 / 16, grid=2, dt=0.1, steps=4, problem="mms")
    sim = LPFEM(cfg)
    for dt in (0.1, 0.1, 0.05, 0.05):
        sim.step(dt)
        st = sim.stats()
        assert max(st["max_rel_residual"]) <= 1e-12, st
    f = sim.fields()
    assert all(np.isfinite(np.ravel(v)).all() for v in f.values())
    sim.close()


@pytest.mark.parametrize("dim,h,H,problem,seed", [(2, 1 / 16, 1 / 4, "mms", None), (2, 1 / 16, 1 / 4, "injection", 2),
                                                  (3, 1 / 8, 1 / 4, "mms", None), (3, 1 / 8, 1 / 4, "injection", 4)])
def test_parity_algorithm1_at_scale_krylov(dim, h, H, problem, seed):
    """SURVEY 8(f) rank 2 at scale: lpfem_opts.algorithm = 1 with H > h solves Algorithm 1 on T_h with
    the fine stage's batched multilevel Krylov kernels on whole-region systems (grid 1, no overlap; H only sets the
    preconditioner's coarsest level) and Newton iterations to the C11 test for the implicit Navier-Stokes step.
    Parity against the oracle's Algorithm 1 (oracle/alg1.py: SuperLU, Picard) at the C20 bar, every step."""
    from oracle import alg1
    from oracle import mesh as M
    from paper_2311_05170_b200 import LPFEM
    dt = 0.1 if problem == "mms" else 0.01
    cfg = I.make_config(dim=dim, H=H, h=h, grid=1, dt=dt, steps=3, problem=problem, seed=seed, overlap=0.0,
                        algorithm=1)
    Gp, Gc = M.region_grids(cfg, "h")
    ora = alg1.Alg1(cfg, Gp, Gc, int(round(H / h)))
    sim = LPFEM(cfg)
    for n in range(cfg["steps"]):
        ora.step()
        sim.step()
        o = {k: np.asarray(v) for k, v in ora.state.items()}
        errs, bad = compare(sim.fields(), o)
        assert not bad, f"step {n + 1}: {errs} {sim.stats()}"
    st = sim.stats()
    assert st["picard_iters"] >= cfg["steps"] and max(st["max_rel_residual"]) <= 1e-12
    sim.close()


@pytest.mark.parametrize("dim,h,dt", [(2, 1 / 16, 0.1), (3, 1 / 4, 0.1)])
def test_parity_algorithm1_on_fine_mesh(dim, h, dt):
    """with H = h the library marches Algorithm 1 on T_h (the traditional
    partitioned scheme the paper compares against).  Parity against the oracle's own Algorithm 1 (oracle/alg1.py),
    C20 bar, every step."""
    from oracle import alg1
    from oracle import mesh as M
    from paper_2311_05170_b200 import LPFEM
    cfg = I.make_config(dim=dim, H=h, h=h, grid=2, dt=dt, steps=3, problem="mms")
    Gp, Gc = M.region_grids(cfg, "h")
    ora = alg1.Alg1(cfg, Gp, Gc, 1)
    sim = LPFEM(cfg)
    for n in range(cfg["steps"]):
        ora.step()
        sim.step()
        o = {k: np.asarray(v) for k, v in ora.state.items()}
        errs, bad = compare(sim.fields(), o)
        assert not bad, f"step {n + 1}: {errs}"
    sim.close()
