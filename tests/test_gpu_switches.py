"""Scheduling-only experiment switches (DESIGN 5.5) leave the result bitwise unchanged.

The switches below change where and when the kernels of a step run (stream priorities, the coarse step's overlap,
the launch order of the systems of a Krylov launch, the gate of the porous PCG behind the GMRES launch), never a
system's arithmetic: cluster sizes, reduction orders and operators are the same.  So the fields after a few steps
must be bit-identical to the default run's (the environment is read once by lpfem_create)."""
import numpy as np
import pytest

import lpfem_inputs as I

pytestmark = pytest.mark.gpu

SWITCHES = ["LPFEM_PCG_PRIO", "LPFEM_NO_PRIO", "LPFEM_NO_OVERLAP", "LPFEM_NO_ORDER", "LPFEM_PCG_UNGATED"]
CASES = {
    "2d-4x4-lognormal": lambda: I.make_config(dim=2, H=1 / 8, h=1 / 32, grid=4, dt=0.01, steps=3,
                                              problem="injection", seed=2),
    "3d-2x2x2": lambda: I.make_config(dim=3, H=1 / 2, h=1 / 4, grid=2, dt=0.1, steps=3, problem="mms"),
}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2311_05170_b200 import build
    build.build()


def _run(cfg):
    from paper_2311_05170_b200 import LPFEM
    sim = LPFEM(cfg)
    for _ in range(cfg["steps"]):
        sim.step()
    f = {k: np.array(v, copy=True) for k, v in sim.fields().items()}
    st = sim.stats()
    sim.close()
    return f, st


@pytest.mark.parametrize("case", list(CASES))
def test_scheduling_switches_are_bitwise_neutral(case, monkeypatch):
    cfg = CASES[case]()
    ref, st0 = _run(cfg)
    for sw in SWITCHES:
        monkeypatch.setenv(sw, "1")
        got, st = _run(cfg)
        monkeypatch.delenv(sw)
        assert st["fine_iters"] == st0["fine_iters"], (sw, st["fine_iters"], st0["fine_iters"])
        for k in ref:
            assert np.array_equal(got[k], ref[k]), (sw, k, float(np.abs(got[k] - ref[k]).max()))
