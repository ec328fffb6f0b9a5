"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import collections
import csv
import sys


def summarise(path, title, out):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        k = r[ki].split("(")[0].replace("void ", "")
        tot[k] += v * scale
        cnt[k] += 1
    T = sum(tot.values())
    with open(out, "w") as f:
        f.write(title + "\n")
        f.write(f"{'kernel':64s} {'launches':>8s} {'total_ms':>12s} {'share':>7s}\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"{k:64s} {cnt[k]:8d} {v:12.3f} {v / T:7.3f}\n")
    print(open(out).read())


if __name__ == "__main__":
    summarise(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1], sys.argv[2])
