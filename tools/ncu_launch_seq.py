"""Print a launch sequence from an ncu launch list (--metrics gpu__time_duration.sum --csv):
one line per kernel launch with its grid and device time, optionally only the last N launches.
Usage: python tools/ncu_launch_seq.py launches.csv [last_n]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, gi, vi, ui = (h.index("Kernel Name"), h.index("Grid Size") if "Grid Size" in h else None,
                  h.index("Metric Value"), h.index("Metric Unit"))
out = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].split("::")[-1]
    t = float(r[vi].replace(",", ""))
    t = t / 1e6 if r[ui] in ("nsecond", "ns") else (t / 1e3 if r[ui] in ("usecond", "us") else t)
    out.append((name[:60], r[gi] if gi is not None else "", t))
last = int(sys.argv[2]) if len(sys.argv) > 2 else len(out)
tot = 0.0
for name, grid, t in out[-last:]:
    tot += t
    print(f"{t:8.3f} ms  {grid:>16s}  {name}")
print(f"{tot:8.3f} ms total over {min(last, len(out))} launches")
