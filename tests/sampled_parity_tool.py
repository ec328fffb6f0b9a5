"""Sampled one-step parity at BASELINE's full sizes, split in two halves so that the slow oracle half (a 3D
Taylor-Hood SuperLU factorisation of a cfg4 box takes ~10 minutes) can run off the GPU box:

    python tests/sampled_parity_tool.py dump CFG N POSITIONS REGIONS OUT.npz     # GPU: the product path
    python tests/sampled_parity_tool.py check OUT.npz LOG                        # CPU: the oracle

dump: runs N steps of config CFG through the C-ABI (LPFEM(cfg), the launch configuration bench.py times) and
stores, for the extended boxes of the sampled positions (comma-separated lexicographic indices) in REGIONS ("p",
"c" or "pc"), the global node indices and the composite values at t_{N-1} (the lagged state, mode B C2) and at
t_N.  No oracle code runs in this half.

check: the oracle (oracle/alg3.py) marches its own coarse trajectory (Step 1) to t_{N-1}, takes the
GPU composite at t_{N-1} on those boxes as the lagged state, solves the sampled subdomains' corrections
 by SuperLU and writes their cores back; the cores must match the GPU composite at t_N
to 1e-9 per field (C20).  Writes a log line per compared (field, position).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import lpfem_inputs as I  # noqa: E402


def _box_nodes(box0, box1, n_cells, vertex=False):
    d = len(n_cells)
    if vertex:
        axes = [np.arange(box0[a], box1[a] + 1) for a in range(d)]
        shape = [k + 1 for k in n_cells]
    else:
        axes = [np.arange(2 * box0[a], 2 * box1[a] + 1) for a in range(d)]
        shape = [2 * k + 1 for k in n_cells]
    grid = np.meshgrid(*axes[::-1], indexing="ij")
    idx = np.zeros(grid[0].shape, dtype=np.int64)
    stride = 1
    for a in range(d):
        idx += grid[d - 1 - a] * stride
        stride *= shape[a]
    return idx.ravel()


def dump(cfgi, n, positions, regions, out):
    from paper_2311_05170_b200 import LPFEM
    cfg = I.config(cfgi)
    sim = LPFEM(cfg)
    for _ in range(n - 1):
        sim.step()
    prev = sim.fields()
    sim.step()
    cur = sim.fields()
    st = sim.stats()
    lay = sim.layout()
    sim.close()
    d = cfg["dim"]
    nf = [int(round(1 / cfg["h"]))] * d
    data = {"cfg": cfgi, "n": n, "positions": np.asarray(positions), "regions": regions,
            "max_rel_residual": np.asarray(st["max_rel_residual"])}
    for L in lay:
        if L["pos"] not in positions or L["region"] not in regions:
            continue
        tag = f"{L['region']}{L['pos']}"
        i2 = _box_nodes(L["box0"], L["box1"], nf)
        data[tag + "_i2"] = i2
        if L["region"] == "p":
            for f in ("pF", "pf", "pm"):
                data[tag + "_prev_" + f] = prev[f][i2]
                data[tag + "_cur_" + f] = cur[f][i2]
        else:
            i1 = _box_nodes(L["box0"], L["box1"], nf, vertex=True)
            data[tag + "_i1"] = i1
            data[tag + "_prev_u"] = prev["u"][:, i2]
            data[tag + "_cur_u"] = cur["u"][:, i2]
            data[tag + "_cur_p"] = cur["p"][i1]
    np.savez_compressed(out, **data)
    print("dumped", out, "max_rel_residual", st["max_rel_residual"])


def check(path, log):
    from gpu_helpers import rel_l2
    from oracle import mesh as M
    from oracle.alg3 import Alg3
    z = np.load(path)
    cfgi, n = int(z["cfg"]), int(z["n"])
    positions = [int(p) for p in z["positions"]]
    regions = str(z["regions"])
    cfg = I.config(cfgi)
    t0 = time.time()
    ora = Alg3(cfg, positions=positions, regions=tuple(regions))
    lexpos = lambda sub: int(M.lex_index(np.asarray(sub.index), np.zeros(cfg["dim"], np.int64), np.asarray(cfg["grid"])))
    for P in ora.P + ora.C:
        P["pos"] = lexpos(P["sub"])
    for _ in range(n - 1):
        ora.coarse.step()
    ora.t_index = n - 1
    # lagged state: the GPU composite at t_{n-1} on the sampled boxes (NaN elsewhere: never read)
    comp = {k: np.full_like(v, np.nan) for k, v in ora.comp.items()}
    for P in ora.P:
        tag = f"p{int(P['pos'])}"
        for f in ("pF", "pf", "pm"):
            comp[f][z[tag + "_i2"]] = z[tag + "_prev_" + f]
    for C in ora.C:
        tag = f"c{int(C['pos'])}"
        comp["u"][:, z[tag + "_i2"]] = z[tag + "_prev_u"]
    ora.comp = comp
    ora.step()
    lines, worst = [], 0.0
    for P in ora.P:
        tag = f"p{int(P['pos'])}"
        i2 = z[tag + "_i2"]
        pos_of = {g: k for k, g in enumerate(i2)}
        idx = P["gidx"][P["own"]]
        sel = np.array([pos_of[g] for g in idx])
        for f in ("pF", "pf", "pm"):
            e = rel_l2(z[tag + "_cur_" + f][sel], ora.comp[f][idx])
            worst = max(worst, e)
            lines.append(f"porous position {P['pos']} field {f}: rel l2 {e:.3e} over {len(idx)} core nodes")
    for C in ora.C:
        tag = f"c{int(C['pos'])}"
        i2, i1 = z[tag + "_i2"], z[tag + "_i1"]
        pos2 = {g: k for k, g in enumerate(i2)}
        pos1 = {g: k for k, g in enumerate(i1)}
        idx = C["gidx"][C["own"]]
        idx1 = C["gidx1"][C["own1"]]
        e = rel_l2(z[tag + "_cur_u"][:, [pos2[g] for g in idx]], ora.comp["u"][:, idx])
        ep = rel_l2(z[tag + "_cur_p"][[pos1[g] for g in idx1]], ora.comp["p"][idx1])
        worst = max(worst, e, ep)
        lines.append(f"conduit position {C['pos']} (Gamma: {C['sub'].box.c0[-1] == 0}) velocity: rel l2 {e:.3e} "
                     f"over {len(idx)} core nodes; pressure: rel l2 {ep:.3e} over {len(idx1)} core vertices")
    head = (f"cfg{cfgi} sampled one-step parity at step {n}: positions {positions} regions {regions}; GPU max rel "
            f"residual {list(z['max_rel_residual'])}; oracle {time.time() - t0:.0f} s (SciPy SuperLU, 1 process)")
    verdict = f"worst {worst:.3e} -> {'PASS' if worst <= 1e-9 else 'FAIL'} (C20 bar 1e-9)"
    txt = "\n".join([head] + lines + [verdict]) + "\n"
    open(log, "w").write(txt)
    print(txt)
    return worst <= 1e-9


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(int(sys.argv[2]), int(sys.argv[3]), [int(p) for p in sys.argv[4].split(",")], sys.argv[5], sys.argv[6])
    else:
        sys.exit(0 if check(sys.argv[2], sys.argv[3]) else 1)
