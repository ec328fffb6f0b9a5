"""Summarise an ncu raw-page CSV (ncu -i REP --page raw --csv): key metrics per kernel launch.

    python tools/ncu_csv.py gpurun_out/NAME_raw.csv [kernel-substring] [min-ms]
"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "local_load_bytes"]


def rows(path):
    r = list(csv.reader(open(path)))
    return r[0], r[1], r[2:]


def main(path, filt=None, min_ms=0.0):
    h, u, data = rows(path)
    ti = h.index("gpu__time_duration.sum")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u[ti], 1.0)
    for r in data:
        name = r[h.index("Kernel Name")]
        if filt and filt not in name:
            continue
        if float(r[ti]) * scale < min_ms:
            continue
        print("==", name[:110])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"   {k:80s} {r[i]:>22s} {u[i]}")


def record(path, kernel, workload, out_txt, desc, min_ms=0.0):
    """Write the summary of the launches of `kernel` (>= min_ms) to out_txt and their mean DRAM bytes per launch to
    profiles/ncu_traffic.json under "kernel@workload" (bench.py's roofline.traffic)."""
    import io
    import json
    import os
    from contextlib import redirect_stdout
    buf = io.StringIO()
    with redirect_stdout(buf):
        main(path, kernel, min_ms)
    open(out_txt, "w").write(desc + "\n" + buf.getvalue())
    h, u, data = rows(path)
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    ti = h.index("gpu__time_duration.sum")
    tsc = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u[ti], 1.0)
    tot, n = 0.0, 0
    for r in data:
        if kernel not in r[h.index("Kernel Name")] or float(r[ti]) * tsc < min_ms:
            continue
        rd = float(r[h.index("dram__bytes_read.sum")]) * sc[u[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")]) * sc[u[h.index("dram__bytes_write.sum")]]
        tot += rd + wr
        n += 1
    tpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    traffic[f"{kernel}@{workload}"] = {"dram_bytes_per_launch": tot / max(n, 1), "source": os.path.basename(out_txt),
                                        "what": desc}
    json.dump(traffic, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "--record":  # --record RAW KERNEL WORKLOAD OUT_TXT DESC [MIN_MS]
        record(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5], sys.argv[6],
               float(sys.argv[7]) if len(sys.argv) > 7 else 0.0)
        sys.exit(0)
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, float(sys.argv[3]) if len(sys.argv) > 3 else 0.0)
