"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals for the LAST pipeline step in the list.

usage: python tools/launch_summary.py launches.csv [first-kernel-of-step-regex]
The step is taken as the suffix starting at the last launch whose name matches
the regex (default: the last k_eg_count, the first kernel of build_topology)."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
L = [(r[ki].split("(")[0].replace("void ", ""), float(r[mi].replace(",", "")), r[ui]) for r in rows[hi + 1:]]
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else r"k_eg_count")
start = max(i for i, (n, _, _) in enumerate(L) if pat.search(n))
step = L[start:]
tot = {}
for n, v, u in step:
    ms = v * scale.get(u, 1e-6)
    c, t = tot.get(n, (0, 0.0))
    tot[n] = (c + 1, t + ms)
S = sum(t for _, t in tot.values())
print(f"step: {len(step)} launches, {S:.3f} ms summed kernel time (ncu: serialised, cold cache)")
print(f"{'kernel':32s} {'launches':>8s} {'ms':>9s} {'share':>7s}")
for n, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:32s} {c:8d} {t:9.3f} {t / S:7.1%}")
