"""Histogram of executed SASS opcodes from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie = h.index("Instructions Executed")
ss = h.index("Warp Stall Sampling (All Samples)")
cnt = collections.Counter()
stall = collections.Counter()
tot = 0
for x in rows[2:]:
    if len(x) <= ie or not x[ie]:
        continue
    op = x[1].split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    cnt[o] += int(x[ie])
    stall[o] += int(x[ss] or 0)
    tot += int(x[ie])
print("total", tot)
for o, c in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print("%-10s %12d %5.1f%%  stall-samples %d" % (o, c, 100 * c / tot, stall[o]))
