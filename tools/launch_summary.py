"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
t, n = defaultdict(float), defaultdict(int)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    v = v / 1e6 if u == "ns" else (v / 1e3 if u == "us" else (v * 1e3 if u == "s" else v))
    name = r[ki].split("(")[0][:64]
    t[name] += v
    n[name] += 1
tot = sum(t.values())
for k, v in sorted(t.items(), key=lambda x: -x[1]):
    print(f"{k:66s} n={n[k]:5d} total_ms={v:10.3f} avg_ms={v / n[k]:9.4f} share={100 * v / tot:6.2f}%")
