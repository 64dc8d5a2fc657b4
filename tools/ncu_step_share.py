"""Per-kernel share of ONE step from an ncu launch list (gpu__time_duration.sum, --csv): the
launches from the last occurrence of the step's first kernel to the end.
Usage: python tools/ncu_step_share.py launches.csv[.gz] first_kernel_substring"""
import csv
import gzip
import sys
from collections import OrderedDict

opener = gzip.open if sys.argv[1].endswith(".gz") else open
rows = [r for r in csv.reader(opener(sys.argv[1], "rt")) if r]
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
ks = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    t = float(r[vi].replace(",", ""))
    t = t / 1e6 if r[ui] in ("nsecond", "ns") else (t / 1e3 if r[ui] in ("usecond", "us") else t)
    ks.append((r[ki].split("(")[0].split("::")[-1], t))
first = max(i for i, (n, _) in enumerate(ks) if sys.argv[2] in n)
step = ks[first:]
tot = sum(t for _, t in step)
agg = OrderedDict()
for n, t in step:
    short = n.split("<")[0]
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += t
print(f"One step from the ncu launch list: {len(step)} launches, {tot:.3f} ms serialised "
      f"(cold-cache, --clock-control none).\n")
print("| kernel | launches | ms | share |")
print("|---|---|---|---|")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {n} | {c} | {t:.3f} | {100 * t / tot:.1f}% |")
