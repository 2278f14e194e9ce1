"""Per-kernel totals of an ncu --csv metrics log (one row per launch x metric)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
h = rows[i]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = defaultdict(lambda: defaultdict(float))
for r in rows[i + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name][r[mi]] += float(r[vi].replace(",", ""))
metrics = sorted({m for d in tot.values() for m in d})
allsum = {m: sum(d[m] for d in tot.values()) for m in metrics}
print("kernel".ljust(34), *[m.split("__")[1][:28].rjust(29) for m in metrics])
for k, d in sorted(tot.items(), key=lambda kv: -kv[1].get(metrics[0], 0)):
    print(k[:34].ljust(34), *[f"{d[m]:29.4g}" for m in metrics])
print("TOTAL".ljust(34), *[f"{allsum[m]:29.4g}" for m in metrics])
