"""Benchmark: fine DOF.steps/s of the local-parallel two-grid FEM hot path (Algorithm 3, arXiv 2311.05170).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl ours|reference]

One "step" = one backward-Euler step of Algorithm 3 through lpfem_step: the coarse step,
every fine subdomain correction (3 porous PCG solves + 1 conduit GMRES solve per subdomain,
with assembly, prolongation, RHS) and the write-back.  Workload: BASELINE.json configs[1]
(2D, H=1/8, h=1/64, 4x4 subdomains, dt=0.05) unless --config says otherwise.  Inputs are synthetic
(the paper's manufactured solution, seeded), resident in HBM when the timed region starts.

Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events on the library's stream;
the L2 is flushed (a 512 MiB write) before every timed step because the cfg1 working set fits in L2.
value = D * K / sum(step times) with D the fine DOF count (3(2N+1)^d + d(2N+1)^d + (N+1)^d).
Multi-GPU: launched by torchrun; ranks own disjoint subdomain positions (weak scaling of the per-GPU
work is not applicable: the problem is fixed, scaling is "strong"); max over ranks.

--impl reference: the CPU oracle (oracle/, SciPy SuperLU per subdomain) timed on this host's cores on a
bounded sample (its first steps of the same workload).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import lpfem_inputs as I  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--alg1", action="store_true",
                    help="Algorithm 1 on T_h (the traditional partitioned scheme, P:356-396): the config with H = h")
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


def cpu_baseline(cfg: dict, budget_s: float = 20.0) -> dict:
    """The oracle as it stands (SciPy SuperLU per subdomain), timed on this host: construction excluded,
    whole steps until ~budget_s of CPU work."""
    from oracle import alg3
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    a = alg3.Alg3(cfg)
    D = I.fine_dofs(cfg)
    n = 0
    t0 = time.perf_counter()
    while n < cfg["steps"] and (n == 0 or time.perf_counter() - t0 < budget_s):
        a.step()
        n += 1
    el = time.perf_counter() - t0
    return {"value": D * n / el, "unit": "fine DOF*steps/s", "cores": 1, "kind": "oracle",
            "sample": f"{cfg['name']}: first {n} of {cfg['steps']} steps ({el:.1f} s), construction excluded, "
                      f"single process (SciPy SuperLU, OPENBLAS_NUM_THREADS=1)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = I.config(args.config)
    D = I.fine_dofs(cfg)
    from oracle import alg3
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    a = alg3.Alg3(cfg)
    budget = 120.0
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        a.step()
        el = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(el)
        if sum(times) > budget or (i + 1) >= cfg["steps"] and False:
            break
        if i + 1 >= cfg["steps"] + args.warmup:
            break
    T = sum(times) if times else float("nan")
    k = len(times)
    value = D * k / T if k else 0.0
    sample = f"{cfg['name']}: {k} timed steps after {args.warmup} warm-up (oracle, SciPy SuperLU, 1 process)"
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": value, "unit": "fine DOF*steps/s",
                      "n_gpus": args.gpus, "steps": k, "warmup": args.warmup,
                      "ms_per_step": 1e3 * T / max(k, 1), "higher_is_better": True, "scaling": "strong",
                      "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": cfg["name"], "dim": cfg["dim"], "H": cfg["H"], "h": cfg["h"],
                                 "grid": cfg["grid"], "dt": cfg["dt"]},
                      "cpu_baseline": {"value": value, "unit": "fine DOF*steps/s", "cores": 1, "kind": "oracle",
                                       "sample": sample},
                      "e2e": {"value": value, "unit": "fine DOF*steps/s", "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}))


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
    if args.alg1:  # H = h: the coarse step is the fine step, the corrections vanish (DESIGN §8(f) rank 2)
        cfg = I.config(args.config, H=cfg["h"], overlap=cfg["h"])
        cfg["name"] += "-alg1"
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
    kr = []
    for k, name in ((0, "k_cg"), (1, "k_gmres")):
        t = st1["t_krylov_ms"][k] - st0["t_krylov_ms"][k]
        b = st1["bytes_krylov"][k] - st0["bytes_krylov"][k]
        n = st1["krylov_launches"][k] - st0["krylov_launches"][k]
        kr.append((t, b, n, name))
    t, b, n, name = max(kr)
    achieved = (b / max(n, 1)) / ((t / max(n, 1)) * 1e-3) / 1e9 if t > 0 else 0.0
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[f"{name}@{cfg['name']}"]
        traffic = tr["dram_bytes_per_launch"]
        traffic_src = tr["source"]
    except Exception:
        traffic_src = None
    roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic, "traffic_source": traffic_src,
            "share_of_step": t / ms if ms > 0 else None,
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
        h2d = (0 if cfg.get("k_mult") is None else np.asarray(cfg["k_mult"]).nbytes) + 8 * 64
        out["e2e"] = {"value": D * args.steps / el, "unit": "fine DOF*steps/s",
                      "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                      "includes": "lpfem_create (setup, assembly) + K x (lpfem_step + lpfem_get_fields to host)",
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
        out["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
