"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch
list per kernel, in first-launch order.

usage: python tools/launch_summary.py LAUNCHES.csv "header line" > profiles/rNN_launch_list_....txt
"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
kn, mn, mv, mu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = OrderedDict()
for r in rows[1:]:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    v = float(r[mv].replace(",", ""))
    u = r[mu]
    us = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000.0 if u in ("ms", "msecond") else v)
    n, t = agg.get(r[kn], (0, 0.0))
    agg[r[kn]] = (n + 1, t + us)
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
for k, (n, t) in agg.items():
    print("%4d launches  avg %10.1f us  total %10.1f us  %s" % (n, t / n, t, k[:120]))
