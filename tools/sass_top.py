"""Top stalled / executed SASS lines from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
body = [x for x in rows[2:] if len(x) > ss]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for x in sorted(body, key=lambda x: -int(x[ss] or 0))[:n]:
    print("%s %-60s exec=%s stall=%s" % (x[0][-5:], x[1].strip()[:60], x[ie], x[ss]))
