"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launches, total/avg device time and share (cold-cache, serialised
per-launch times: compare SHARES, not absolutes)."""
import collections
import csv
import sys

path = sys.argv[1]
skip = sys.argv[2:]  # kernel-name substrings to exclude (e.g. harness-only kernels)
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    if any(s in name for s in skip):
        continue
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(t for _, t in agg.values())
print(f"# {path}: {sum(n for n, _ in agg.values())} launches, {tot:.1f} us total"
      + (f" (excluding {', '.join(skip)})" if skip else ""))
print(f"{'kernel':44s} {'launches':>8s} {'total_us':>11s} {'share':>6s} {'avg_us':>8s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {n:8d} {t:11.1f} {100 * t / tot:5.1f}% {t / n:8.2f}")
