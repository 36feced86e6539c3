"""Per-kernel mean of each metric in an ncu --csv launch list (several --metrics)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0][:64]][f"{r[mi]} [{r[ui]}]"].append(float(r[vi].replace(",", "")))
for k, d in agg.items():
    if len(sys.argv) > 2 and sys.argv[2] not in k:
        continue
    print(k)
    for m, v in d.items():
        print(f"    {m:40s} n={len(v):4d} mean={sum(v) / len(v):14.1f}")
