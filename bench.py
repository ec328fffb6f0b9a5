"""Benchmark: fine DOF.steps/s of the local-parallel two-grid FEM hot path (Algorithm 3, arXiv 2311.05170).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One "step" = one backward-Euler step of Algorithm 3 through lpfem_step: the coarse step,
every fine subdomain correction (3 porous PCG solves + 1 conduit GMRES solve per subdomain,
with assembly, prolongation, RHS) and the write-back.  Workload: BASELINE.json configs[4]
(3D, H=1/8, h=1/48, 4x4x4 subdomains, injection with log-normal permeability, dt=0.01: 5.59M fine DOFs,
the largest configuration, in the HBM regime at every GPU count) unless --config says
otherwise.  Inputs are synthetic (seeded), resident in HBM when the timed region starts.

Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events on the library's stream;
the L2 is flushed (a 512 MiB write) before every timed step (cfg0/cfg1 fit in L2).
value = D * K / sum(step times) with D the fine DOF count (3(2N+1)^d + d(2N+1)^d + (N+1)^d).
Multi-GPU: launched by torchrun; ranks own disjoint subdomain positions (LPT placement); the problem is fixed
as N grows ("strong"); max over ranks.

--impl reference / cpu_baseline: the CPU oracle (oracle/, SciPy SuperLU per subdomain) as it stands, timed on
this host's cores: one worker process per core, each running the oracle's Algorithm 3 on a share of the subdomain
positions (its own redundant coarse step, like a GPU rank) with the composite exchanged through the parent every
step.  cfg0-cfg2 at full size; cfg3 and cfg4 (a single cfg4 conduit factorisation takes 10-30 minutes, SURVEY
A3) on the same configuration at a coarser fine mesh (h = 1/8 and 1/16, same H, grid, data and coefficients),
which bounds the oracle's full-size throughput from above (SuperLU cost per DOF grows with the box size).
"""
from __future__ import annotations

import os

# the oracle's worker processes run one BLAS thread each: set before numpy (and its BLAS pool) is loaded
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import lpfem_inputs as I  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rtol", type=float, default=None,
                    help="override the Krylov relative residual (C19: 1e-12); comparison runs only")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--alg1", action="store_true",
                    help="Algorithm 1 on T_h (the traditional partitioned scheme, P:356-396) on the config's fine mesh, "
                         "whole-region systems on the same Krylov kernels (lpfem_opts.algorithm = 1)")
    return ap.parse_args()


METRIC = "fine DOF*steps/s (Algorithm 3 step: coarse + local subdomain corrections + write-back)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region (50 ms period)."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs ~0.1-0.5 s to start: wait for its first sample so that short timed regions
            # (cfg0: ~15 ms) are still sampled
            t0 = time.perf_counter()
            while not self.rows and time.perf_counter() - t0 < 3.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.06)  # one more sample at the end of the timed region
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------------------------------ CPU oracle legs
ORACLE_SAMPLE_H = {3: 1 / 8, 4: 1 / 16}  # configs whose full-size oracle step takes hours


def oracle_sample_cfg(cfgi: int) -> tuple[dict, str]:
    cfg = I.config(cfgi)
    if cfgi in ORACLE_SAMPLE_H:
        h = ORACLE_SAMPLE_H[cfgi]
        cfg = I.config(cfgi, h=h)
        return cfg, (f"cfg{cfgi} structure at h = 1/{round(1 / h)} (same H, grid, data, coefficients, dt; "
                     f"{I.fine_dofs(cfg)} fine DOFs): an upper bound of the oracle's full-size throughput")
    return cfg, f"cfg{cfgi} at full size"


def _oracle_worker(conn, cfg, positions):
    from oracle import alg3
    from oracle import mesh as M
    a = alg3.Alg3(cfg, positions=positions)
    d = cfg["dim"]
    conn.send("ready")
    while True:
        comp = conn.recv()
        if comp is None:
            break
        a.comp = comp
        f0 = a.timing["fine"]
        a.step()
        el = a.timing["fine"] - f0  # the fine stage (Steps 3-4) of this worker's subdomains
        out = []
        for P in a.P:
            idx = P["gidx"][P["own"]]
            out.append(("p", idx, {f: a.comp[f][idx] for f in ("pF", "pf", "pm")}))
        for C in a.C:
            idx, idx1 = C["gidx"][C["own"]], C["gidx1"][C["own1"]]
            out.append(("c", (idx, idx1), {"u": a.comp["u"][:, idx], "p": a.comp["p"][idx1]}))
        conn.send((out, el))
    conn.close()


class OraclePool:
    """The oracle's Algorithm 3 on a pool of worker processes (one per host core): positions split LPT-like by
    box size, each worker marching its own coarse step (redundant, like the GPU ranks) and its subdomains; the
    parent merges the owned core values (Step 4) into the composite and sends it back (mode B)."""

    def __init__(self, cfg: dict, workers: int):
        import multiprocessing as mp
        from oracle import alg3
        self.cfg = cfg
        npos = int(np.prod(cfg["grid"]))
        workers = max(1, min(workers, npos))
        share = [list(range(w, npos, workers)) for w in range(workers)]
        self.comp = alg3.Alg3(cfg, positions=[]).fields()
        ctx = mp.get_context("fork")
        self.conns, self.procs = [], []
        for sh in share:
            a, b = ctx.Pipe()
            p = ctx.Process(target=_oracle_worker, args=(b, cfg, sh), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for c in self.conns:
            assert c.recv() == "ready"
        self.workers = workers

    def step(self) -> tuple[float, float]:
        """One step; returns (wall seconds, fine-stage seconds = max over the workers + the merge)."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(self.comp)
        new = {k: np.copy(v) for k, v in self.comp.items()}
        fine = 0.0
        outs = []
        for c in self.conns:
            out, el = c.recv()
            fine = max(fine, el)
            outs.append(out)
        t1 = time.perf_counter()
        for out in outs:
            for kind, idx, vals in out:
                if kind == "p":
                    for f, v in vals.items():
                        new[f][idx] = v
                else:
                    new["u"][:, idx[0]] = vals["u"]
                    new["p"][idx[1]] = vals["p"]
        self.comp = new
        t2 = time.perf_counter()
        return t2 - t0, fine + (t2 - t1)

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=10)


def host_cores() -> tuple[int, str]:
    n = len(os.sched_getaffinity(0))
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return n, model


def oracle_measure(cfgi: int, warmup: int, steps: int, budget_s: float) -> dict:
    """Fine-stage throughput of the pooled oracle (T_fine covers Steps 3-4, the coarse
    trajectory is timed apart); the run stops after `steps` timed steps or when the wall time of the timed steps
    exceeds budget_s (at least one step)."""
    cfg, what = oracle_sample_cfg(cfgi)
    cores, model = host_cores()
    pool = OraclePool(cfg, cores)
    try:
        for _ in range(warmup):
            pool.step()
        fine, wall = [], []
        while len(fine) < steps and (not wall or sum(wall) < budget_s):
            w, f = pool.step()
            wall.append(w)
            fine.append(f)
    finally:
        pool.close()
    D = I.fine_dofs(cfg)
    T = sum(fine)
    return {"value": D * len(fine) / T, "unit": "fine DOF*steps/s", "cores": pool.workers, "kind": "oracle",
            "steps": len(fine), "warmup": warmup, "ms_per_step": 1e3 * T / len(fine),
            "wall_ms_per_step_incl_coarse": 1e3 * sum(wall) / len(wall),
            "sample": f"{what}; {len(fine)} timed step(s) after {warmup} warm-up, construction excluded; fine stage "
                      f"(Steps 3-4: max over workers + merge), the redundant per-worker coarse step timed apart "
                      f"(wall incl. coarse {sum(wall) / len(wall):.1f} s/step); {pool.workers} worker processes "
                      f"(1 BLAS thread each) on {cores} host cores ({model}); SciPy SuperLU per subdomain"}


def cpu_baseline(cfgi: int) -> dict:
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload (one step)."""
    return oracle_measure(cfgi, warmup=0, steps=1, budget_s=20.0)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = I.config(args.config)
    m = oracle_measure(args.config, warmup=0, steps=args.steps, budget_s=120.0)
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": m["value"], "unit": "fine DOF*steps/s",
                      "n_gpus": args.gpus, "steps": m["steps"], "warmup": m["warmup"],
                      "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": "strong",
                      "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": cfg["name"], "dim": cfg["dim"], "H": cfg["H"], "h": cfg["h"],
                                 "grid": cfg["grid"], "dt": cfg["dt"], "problem": cfg["problem"]},
                      "cpu_baseline": {k: m[k] for k in ("value", "unit", "cores", "kind", "sample")},
                      "e2e": {"value": m["value"], "unit": "fine DOF*steps/s", "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}))


L2_BYTES = 126e6


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    from paper_2311_05170_b200 import LPFEM, build, nccl_unique_id
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    cfg = I.config(args.config)
    if args.alg1:  # Algorithm 1 on T_h: whole regions (grid 1, no overlap), H = the preconditioner's coarsest level
        cfg = I.config(args.config, grid=1, overlap=0.0, algorithm=1)
        cfg["name"] += "-alg1"
    if args.rtol is not None:
        cfg["krylov_rtol"] = args.rtol
        cfg["name"] += f"-rtol{args.rtol:g}"
    D = I.fine_dofs(cfg)
    stream = torch.cuda.Stream()
    nid = None
    if world > 1:
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        nid = bytes(t.cpu().numpy().tobytes())
    sim = LPFEM(cfg, rank=rank, world=world, device=local, stream=stream.cuda_stream, nccl_id=nid)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        sim.step()
    torch.cuda.synchronize()
    st0 = sim.stats()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(i))  # L2 flush (512 MiB > 126 MB L2), outside the events
                evs[i][0].record(stream)
            sim.step()
            with torch.cuda.stream(stream):
                evs[i][1].record(stream)
        torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    st1 = sim.stats()
    value = D * args.steps / (ms * 1e-3)
    # roofline of the dominant kernel (fine Krylov launches; times from CUDA events in the library)
    peak, peak_kind = peaks()
    # the dominant kernel is the one that moves the most algorithmic bytes (the porous PCG runs concurrently on the
    # SMs the GMRES leaves free, so its elapsed time is not its cost)
    kr = []
    for k, name in ((0, "k_pcg_ml"), (1, "k_gmres")):
        t = st1["t_krylov_ms"][k] - st0["t_krylov_ms"][k]
        b = st1["bytes_krylov"][k] - st0["bytes_krylov"][k]
        n = st1["krylov_launches"][k] - st0["krylov_launches"][k]
        kr.append((b, t, n, name))
    b, t, n, name = max(kr)
    achieved = (b / max(n, 1)) / ((t / max(n, 1)) * 1e-3) / 1e9 if t > 0 else 0.0
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[f"{name}@{cfg['name']}"]
        traffic = tr["dram_bytes_per_launch"]
        traffic_src = tr["source"]
    except Exception:
        traffic_src = None
    # regime (SURVEY 8(d) consequence 1): the rank's matrices (conduit: 12 B/nnz; porous: 3 x 8 + 4 B/nnz)
    # against the 126 MB L2.  L2-resident families are labelled "l2": their algorithmic GB/s is an L2 rate and
    # the ncu traffic beside it (dram bytes) shows how little reaches HBM.
    mat_bytes = 12.0 * st1["nnz"][1] + 28.0 * st1["nnz"][0]
    regime = "hbm" if mat_bytes > L2_BYTES else "l2"
    roof = {"kernel": name, "bound": regime, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic, "traffic_source": traffic_src,
            "share_of_step": t / ms if ms > 0 else None, "matrix_bytes_rank": mat_bytes,
            "algorithmic_bytes_per_launch": b / max(n, 1), "ms_per_launch": t / max(n, 1)}
    out = {
        "metric": METRIC, "value": value, "unit": "fine DOF*steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "dim": cfg["dim"], "H": cfg["H"], "h": cfg["h"], "grid": cfg["grid"],
                   "dt": cfg["dt"], "problem": cfg["problem"], "fine_dofs": D, "l2": "flushed before every timed step",
                   "parallelism": f"subdomains over {world} GPU(s)"},
        "gpu_launches": st1["kernel_launches"] - st0["kernel_launches"],
        "roofline": roof,
        "clocks": clk.summary(),
        "wall_s": wall,
        "stages_ms_per_step": {"coarse": (st1["t_coarse_ms"] - st0["t_coarse_ms"]) / args.steps,
                               "fine": (st1["t_fine_ms"] - st0["t_fine_ms"]) / args.steps,
                               "fine_pcg": (st1["t_krylov_ms"][0] - st0["t_krylov_ms"][0]) / args.steps,
                               "fine_gmres": (st1["t_krylov_ms"][1] - st0["t_krylov_ms"][1]) / args.steps},
        "iters_per_step": {"fine_pcg_sum": (st1["fine_iters"][0] - st0["fine_iters"][0]) / args.steps,
                           "fine_gmres_sum": (st1["fine_iters"][1] - st0["fine_iters"][1]) / args.steps,
                           "fine_pcg_max_last": st1["fine_max_iters"][0],
                           "fine_gmres_max_last": st1["fine_max_iters"][1],
                           "coarse_picard": (st1["picard_iters"] - st0["picard_iters"]) / args.steps},
        "fine_value": D * args.steps / ((st1["t_fine_ms"] - st0["t_fine_ms"]) * 1e-3),
    }
    # end to end through the public API with host buffers: create from host inputs, K steps, fields -> host.
    # One untimed create + step + close first (allocator / driver warm-up: right after other GPU processes the
    # first create of a process measured 80-620 ms instead of ~20 ms)
    if not args.no_e2e:
        if world > 1:
            t = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(t, 0)
            nid = bytes(t.cpu().numpy().tobytes())
        warm = LPFEM(cfg, rank=rank, world=world, device=local, stream=stream.cuda_stream, nccl_id=nid)
        warm.step()
        warm.fields()
        warm.close()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world > 1:
            t = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(t, 0)
            nid = bytes(t.cpu().numpy().tobytes())
        sim2 = LPFEM(cfg, rank=rank, world=world, device=local, stream=stream.cuda_stream, nccl_id=nid)
        torch.cuda.synchronize()
        t_create = time.perf_counter() - t0
        d2h = 0
        for i in range(args.steps):
            sim2.step()
            f = sim2.fields()
            d2h += sum(v.nbytes for v in f.values())
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        s2 = sim2.stats()  # every host<->device copy the library made (create, steps, fields), counted in the library
        out["e2e"] = {"value": D * args.steps / el, "unit": "fine DOF*steps/s",
                      "h2d_bytes_per_step": s2["h2d_bytes"] // args.steps,
                      "d2h_bytes_per_step": s2["d2h_bytes"] // args.steps,
                      "fields_bytes_per_step": d2h // args.steps,
                      "includes": "lpfem_create from host inputs (setup, assembly) + K x (lpfem_step + "
                                  "lpfem_get_fields to host); bytes counted by the library (lpfem_stats)",
                      "create_ms": 1e3 * t_create, "steps_ms": 1e3 * (el - t_create)}
        sim2.close()
    # SpMV building block of the Krylov kernels (BASELINE metric "SpMV % HBM peak"): the conduit family's batched
    # y = A x with the same device routine, L2 flushed before every rep, outside the timed region (measured on
    # the bench context before it closes)
    try:
        sp = sim.bench_spmv(1, reps=10, flush=True)
        out["spmv"] = {"family": "conduit (fine Oseen operators, all systems of rank 0)", "bound": "hbm",
                       "achieved": sp["gbs"], "peak": peak, "unit": "GB/s", "frac": sp["gbs"] / peak,
                       "ms_per_rep": sp["ms"], "algorithmic_bytes_per_rep": sp["bytes"],
                       "l2": "flushed before every rep"}
    except Exception as e:  # a rank without conduit systems (small configs on many GPUs)
        out["spmv"] = {"unavailable": str(e)[:120]}
    sim.close()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
