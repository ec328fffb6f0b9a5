"""The multi-rank path executed on one GPU (VERDICT r1 "What's missing" 3).

All `world` ranks are contexts of this process (LPFEM_TRANSPORT_LOCAL) stepped together by lpfem_step_group:
the same LPT placement, halo plan (csrc/halo.h), pack / unpack kernels, shadow-composite commit and gather to the
root as the NCCL transport -- only the transfer itself is a cudaMemcpyPeerAsync out of the peer's packed send
buffer instead of ncclSend/ncclRecv.  The ranks' kernels never wait on each other inside a launch (dependencies
are stream events between phases).

* world 2 and 4 against the oracle (C20) and against world 1, mode B (the halo exchange carries the lagged
  state of the overlaps, C2) and mode A (no exchange needed);
* world_invariant: bitwise identical fields for world 1, 2, 4;
* an ENOCONV on one rank commits nothing on any rank.
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


def _run(cfg, world, steps, **kw):
    from paper_2311_05170_b200 import LPFEM, LocalGroup
    sim = LPFEM(cfg, **kw) if world == 1 else LocalGroup(cfg, world, **kw)
    out = []
    for _ in range(steps):
        sim.step()
        out.append(sim.fields())
    st = sim.stats()
    sim.close()
    return out, st


CASES = {
    "cfg0": lambda: I.config(0, steps=3),
    "2d-4x4-lognormal": lambda: I.make_config(dim=2, H=1 / 8, h=1 / 32, grid=4, dt=0.01, steps=3,
                                              problem="injection", seed=2),
    "3d-2x2x2": lambda: I.make_config(dim=3, H=1 / 2, h=1 / 4, grid=2, dt=0.1, steps=2, problem="mms"),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("world", [2, 4])
def test_world_matches_oracle_and_world1(case, world):
    from oracle import alg3
    cfg = CASES[case]()
    ora = alg3.Alg3(cfg)
    got, _ = _run(cfg, world, cfg["steps"])
    one, _ = _run(cfg, 1, cfg["steps"])
    for n in range(cfg["steps"]):
        ora.step()
        errs, bad = compare(got[n], ora.fields())
        assert not bad, (n + 1, errs)
        errs1, bad1 = compare(got[n], one[n], tol=1e-10)
        assert not bad1, (n + 1, errs1)


@pytest.mark.parametrize("world", [2, 4])
def test_world_mode_a(world):
    cfg = I.config(0, steps=3, lag_mode="subdomain")
    from oracle import alg3
    ora = alg3.Alg3(cfg)
    got, _ = _run(cfg, world, 3)
    for n in range(3):
        ora.step()
        errs, bad = compare(got[n], ora.fields())
        assert not bad, (n + 1, errs)


@pytest.mark.parametrize("case", ["cfg0", "3d-2x2x2"])
def test_world_invariant_bitwise(case):
    cfg = CASES[case]()
    ref, _ = _run(cfg, 1, cfg["steps"], world_invariant=True)
    for world in (2, 4):
        got, _ = _run(cfg, world, cfg["steps"], world_invariant=True)
        for n in range(cfg["steps"]):
            for k in ref[n]:
                assert np.array_equal(np.asarray(got[n][k]), np.asarray(ref[n][k])), (world, n + 1, k)


def test_world_enoconv_on_one_rank_commits_nothing():
    from paper_2311_05170_b200 import LocalGroup, LPFEMError
    cfg = I.config(0, steps=3)
    g = LocalGroup(cfg, 2)
    g.step()
    before = g.fields()
    g.ranks[1].inject_fault(1, 1)
    with pytest.raises(LPFEMError) as e:
        g.step()
    assert e.value.status == 4
    assert all(r.stats()["steps"] == 1 for r in g.ranks)
    after = g.fields()
    assert all(np.array_equal(np.asarray(after[k]), np.asarray(before[k])) for k in before)
    g.ranks[1].inject_fault(1, 0)
    g.step()
    assert all(r.stats()["steps"] == 2 for r in g.ranks)
    g.close()
