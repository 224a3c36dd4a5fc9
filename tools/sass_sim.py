"""Static in-order issue model of a straight-line SASS window (one warp alone
on its scheduler): estimates cycles for the window from register dependencies.

usage: cuobjdump -sass X.o > x.sass; python tools/sass_sim.py x.sass FUNC_SUBSTR START END
Latencies (B200, measured where noted): fp64 ops 8 (tools/dadd_latency.cu),
fp64 pipe one warp instruction per 2 cycles, ALU 4, IMAD 5, LDS 30.
"""
import re
import sys


def regs(tok):
    out = []
    for m in re.finditer(r"\bR(\d+)(\.64)?\b", tok):
        out.append(int(m.group(1)))
    return out


def parse(line):
    line = re.sub(r"@!?U?P\d+\s+", "", line)
    op, _, rest = line.partition(" ")
    ops = [o.strip() for o in rest.split(",")] if rest else []
    base = op.split(".")[0]
    wide = base in ("DADD", "DMUL", "DFMA") or ".64" in op or ".WIDE" in op
    w128 = ".128" in op
    dst, src = [], []
    if base in ("STS", "STG", "BRA", "BSYNC", "BSSY", "SYNCS", "UTMALDG", "UBLKCP", "WARPSYNC", "NOP", "EXIT"):
        for o in ops:
            src += regs(o)
    elif ops:
        d = regs(ops[0])
        if d and not ops[0].startswith("["):
            n = 4 if w128 else (2 if wide else 1)
            dst = list(range(d[0], d[0] + n))
        for o in ops[1:]:
            r = regs(o)
            for x in r:
                src.append(x)
                if base in ("DADD", "DMUL", "DFMA") and not o.startswith("["):
                    src.append(x + 1)
    return base, dst, src


LAT = {"DADD": 8, "DMUL": 8, "DFMA": 8, "LDS": 30, "IMAD": 5, "LDG": 400}


def main():
    path, sub, a, b = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    fn, ins = None, []
    for l in open(path):
        m = re.search(r"Function : (\S+)", l)
        if m:
            fn = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(.*?);", l)
        if m and fn and sub in fn:
            ins.append(m.group(1).strip())
    win = ins[a:b]
    ready = {}
    t = 0
    fp64_free = 0
    stall_by = {}
    for s in win:
        base, dst, src = parse(s)
        issue = t + 1
        for r in src:
            issue = max(issue, ready.get(r, 0))
        if base in ("DADD", "DMUL", "DFMA"):
            issue = max(issue, fp64_free)
            fp64_free = issue + 2
        stall_by[base] = stall_by.get(base, 0) + (issue - t - 1)
        t = issue
        lat = LAT.get(base, 4)
        for r in dst:
            ready[r] = t + lat
    print("%d instructions, %d cycles, IPC %.2f" % (len(win), t, len(win) / max(t, 1)))
    print("stall cycles by waiting op:", sorted(stall_by.items(), key=lambda kv: -kv[1])[:6])


main()
