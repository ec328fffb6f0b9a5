"""The C-ABI's error and time contracts on the GPU (include/lpfem.h, lpfem_step):

* LPFEM_ENOCONV commits nothing (SPEC.md:357 SolverFailure; SURVEY 5 fault injection by a max_iter cap):
  fields() and stats().steps stay at t_n, and the retried step reproduces the uninterrupted trajectory.
* C18 with a dt change: t_{n+1} = t_b + (n+1-n_b) dt, checked through the Dirichlet data, which the composite
  carries exactly on the physical boundary (C5: e = I_h g(t_{n+1}) - P u_H^{n+1} there).
"""
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


def _same(a, b):
    return all(np.array_equal(np.asarray(a[k]), np.asarray(b[k])) for k in a)


@pytest.mark.parametrize("family,lag", [(1, "composite"), (0, "composite"), (1, "subdomain"), (0, "subdomain")])
def test_fine_enoconv_commits_nothing_and_retry_matches(family, lag):
    from paper_2311_05170_b200 import LPFEM, LPFEMError
    cfg = I.config(0, lag_mode=lag)
    ref = LPFEM(cfg)
    for _ in range(3):
        ref.step()
    want = ref.fields()
    ref.close()
    sim = LPFEM(cfg)
    sim.step()
    sim.step()
    before, st0 = sim.fields(), sim.stats()
    sim.inject_fault(family, 1)
    for _ in range(2):  # repeated failures leave the state alone too
        with pytest.raises(LPFEMError) as e:
            sim.step()
        assert e.value.status == 4  # LPFEM_ENOCONV
        assert _same(sim.fields(), before)
        assert sim.stats()["steps"] == st0["steps"] == 2
    sim.inject_fault(family, 0)
    sim.step()
    assert sim.stats()["steps"] == 3
    errs, bad = compare(sim.fields(), want, tol=1e-10)
    assert not bad, errs
    sim.close()


def test_coarse_enoconv_commits_nothing():
    """max_iter = 1 for every solve: the coarse porous PCG of Step 1 fails first; the initial state stays."""
    from paper_2311_05170_b200 import LPFEM, LPFEMError
    cfg = I.config(0)
    sim = LPFEM(cfg, max_iter=1)
    before = sim.fields()
    with pytest.raises(LPFEMError) as e:
        sim.step()
    assert e.value.status == 4
    assert "coarse" in str(e.value)
    assert _same(sim.fields(), before)
    assert sim.stats()["steps"] == 0
    sim.close()


def test_dt_change_time_levels():
    """dt = 0.1, 0.1, 0.05, 0.05: the data of the steps are evaluated at t = 0.1, 0.2, 0.25, 0.3 (C18 within each
    constant-dt segment), seen on the Dirichlet nodes of both regions, which carry I_h g(t_{n+1}) exactly (C5)."""
    from oracle import mesh as M
    from oracle.mms import Problem
    from paper_2311_05170_b200 import LPFEM
    cfg = I.config(0)
    pr = Problem(cfg)
    Gp, Gc = M.region_grids(cfg, "h")
    bp, bc = M.Box(Gp, (0, 0), Gp.n), M.Box(Gc, (0, 0), Gc.n)
    dir_p = bp.classes(whole_region=True) == M.DIR
    dir_c = bc.classes(whole_region=True) == M.DIR
    Xp, Xc = Gp.coords(bp.node_g), Gc.coords(bc.node_g)
    sim = LPFEM(cfg)
    t = 0.0
    for dt in (0.1, 0.1, 0.05, 0.05):
        sim.step(dt)
        t += dt
        f = sim.fields()
        for k in ("pF", "pf", "pm"):
            ex = pr.porous(k, Xp[dir_p], t)
            assert np.abs(f[k][dir_p] - ex).max() <= 1e-12 * max(1.0, np.abs(ex).max()), (k, t)
        exu = pr.velocity(Xc[dir_c], t)
        assert np.abs(f["u"][:, dir_c] - exu).max() <= 1e-12 * max(1.0, np.abs(exu).max()), t
        assert max(sim.stats()["max_rel_residual"]) <= 1e-12
    sim.close()
