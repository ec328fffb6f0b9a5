"""Aggregate ncu source-page stall samples and executed instructions per CUDA source line.
    python tools/ncu_lines.py report.ncu-rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = []; fname = "?"; hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] == "Function Name": continue
    if r[2] != "-": continue  # sass rows
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ins = float(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    agg.append((s, ins, fname, r[0], r[1]))
ts = sum(a[0] for a in agg) or 1; ti = sum(a[1] for a in agg) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.3g}")
for s, ins, f, ln, src in sorted(agg, key=lambda a: -a[0])[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*ins/ti:5.1f}% ins  {f}:{ln:<5} {src.strip()[:100]}")
