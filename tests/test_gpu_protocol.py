"""SURVEY 8(f) rank 3, the paper's convergence protocol on the GPU (Tables 1-2): Example 1 with all
coefficients 1, 2x2 subdomains per region with the fixed extension 1/4, h = H^2, dt = h^2, T = 1, at
h = 1/4, 1/16, 1/64 (the paper's fourth row, h = 1/256, is 65536 steps of a 256^2 mesh: left out).  Elements:
Taylor-Hood P2-P1 and P2 porous pressures (reading C1) instead of the paper's MINI / P1, so the paper's numbers
are context only; what is checked is the paper's claim that Algorithm 3 keeps Algorithm 1's accuracy (T1 vs T2)
and that the errors converge.  Norms: tests/protocol_norms.py (piecewise norms of P:1465-1475)."""
import json
import math
import os

import pytest

import protocol_norms as PN

pytestmark = pytest.mark.gpu
# Levels run: h = 1/4, 1/16 by default (20 s on a B200); LPFEM_PROTOCOL_LEVELS=0,1,2 adds h = 1/64 (4096 steps per
# scheme, +3.5 min), the run whose table is committed as profiles/r02_protocol_ex1_th.json (DESIGN 7).
LEVELS = tuple(int(x) for x in os.environ.get("LPFEM_PROTOCOL_LEVELS", "0,1").split(","))
# porous columns of Algorithm 3 against Algorithm 1's at the finest level run: within 2x at h = 1/64; at h = 1/16
# the coarse term H^3 = 1/64 still shows in |||p_m|||_0 (measured 3.0x), so the bound there is 3.5x
POROUS_FACTOR = {1: 3.5, 2: 2.0}


@pytest.fixture(scope="module")
def runs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2311_05170_b200 import LPFEM
    out = {}
    for alg in (3, 1):
        for lev in LEVELS:
            cfg = PN.protocol_config(lev, algorithm=alg)
            sim = LPFEM(cfg)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            ev0.record()
            for _ in range(cfg["steps"]):
                sim.step()
            ev1.record()
            torch.cuda.synchronize()
            f = sim.fields()
            st = sim.stats()
            sim.close()
            e = PN.table_errors(cfg, f)
            e["gpu_s"] = ev0.elapsed_time(ev1) / 1e3
            e["steps"] = cfg["steps"]
            e["fine_iters"] = st["fine_iters"]
            out[(alg, lev)] = e
    rows = [{"algorithm": a, "h": PN.protocol_config(l)["h"], "H": PN.protocol_config(l)["H"], **out[(a, l)]}
            for (a, l) in sorted(out)]
    print("PROTOCOL_TABLE " + json.dumps(rows))
    if os.environ.get("LPFEM_PROTOCOL_OUT"):
        with open(os.environ["LPFEM_PROTOCOL_OUT"], "w") as fh:
            json.dump(rows, fh, indent=1)
    return out


COLS = ("u_1", "pF_1", "pf_0", "pf_1", "pm_0", "pm_1")


def _rate(e0, e1, h0, h1):
    return math.log(e0 / e1) / math.log(h0 / h1)


def test_local_parallel_against_the_traditional_scheme(runs):
    """T1 vs T2 with Taylor-Hood elements.  Theorem P:1478-1494 bounds Algorithm 3's error by
    Delta t + h^r + H^(r+1) (times 1 + Delta t^(-1/2) in H1); with r = 2 and the paper's scaling h = H^2 the coarse
    term H^3 = h^1.5 exceeds Algorithm 1's h^2, so only the porous errors are expected to match Algorithm 1's at the
    finest level (the paper's MINI/P1 has r = 1, where H^2 = h matches): porous columns within 2x of Algorithm 1's
    at h = 1/64 (3.5x at h = 1/16, POROUS_FACTOR);
    the velocity gap |||u|||_1(Alg 3) - |||u|||_1(Alg 1) shrinks from level to level."""
    lev = LEVELS[-1]
    for k in COLS[1:]:
        assert runs[(3, lev)][k] <= POROUS_FACTOR[lev] * runs[(1, lev)][k], (lev, k, runs[(3, lev)][k], runs[(1, lev)][k])
    gaps = [runs[(3, l)]["u_1"] - runs[(1, l)]["u_1"] for l in LEVELS]
    print("velocity H1 gap Alg3 - Alg1 per level", gaps)
    assert all(b < a for a, b in zip(gaps[:-1], gaps[1:])), gaps


def test_errors_converge(runs):
    """Every column decreases from level to level, with an observed rate in h of at least 1 between the two finest
    levels (the paper's MINI/P1 H1 rate, Table 1)."""
    h = [PN.protocol_config(l)["h"] for l in LEVELS]
    for alg in (3, 1):
        for k in COLS:
            for a, b in zip(LEVELS[:-1], LEVELS[1:]):
                assert runs[(alg, b)][k] < runs[(alg, a)][k], (alg, k, a, b)
            r = _rate(runs[(alg, LEVELS[-2])][k], runs[(alg, LEVELS[-1])][k], h[-2], h[-1])
            print(f"algorithm {alg} rate {k}: {r:.2f}")
            assert r >= 1.0, (alg, k, r)
