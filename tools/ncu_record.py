"""Record an ncu --set full report under profiles/: key metrics per kernel launch (text) and, for bench.py's
roofline, the DRAM traffic per launch of each kernel (profiles/ncu_traffic.json).

    python tools/ncu_record.py gpurun_out/prof.ncu-rep profiles/r01_ncu_gmres_cfg1.txt "description" cfg1
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, out, desc, workload):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    lines = [desc, f"report: {os.path.basename(rep)} (ncu --set full --clock-control none --import-source on)", ""]
    traffic = {}
    tpath = os.path.join(os.path.dirname(out), "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").split("<")[0].replace("lp::", "")
        lines.append(f"== {name[:120]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"   {k:75s} {r[i]:>18s} {u[i]}")
        try:
            rd = float(r[h.index("dram__bytes_read.sum")]) * SCALE[u[h.index("dram__bytes_read.sum")]]
            wr = float(r[h.index("dram__bytes_write.sum")]) * SCALE[u[h.index("dram__bytes_write.sum")]]
            if rd + wr == rd + wr:  # not NaN
                traffic[f"{short}@{workload}"] = {"dram_bytes_per_launch": rd + wr, "source": os.path.basename(out),
                                                  "what": desc}
        except (ValueError, KeyError):
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4])
