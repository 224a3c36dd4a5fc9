"""Top SASS instructions by warp-stall samples from an ncu source-page CSV.

usage: ncu -i REP --page source --csv --kernel-name regex:NAME --print-source sass > s.csv
       python tools/sass_stalls.py s.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
data = []
for r in rows:
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    i = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        data.append((float(r[i]), r[0], r[1]))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print("total samples %d, instructions %d" % (tot, len(data)))
for k, (v, a, src) in enumerate(data):
    data[k] = (v, k, a, src)
for v, k, a, src in sorted(data, key=lambda d: -d[0])[:n]:
    print("%7d %5.1f%%  #%-5d %s" % (v, 100 * v / max(tot, 1), k, src.strip()[:100]))
