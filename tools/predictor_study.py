"""Bytes per entry of candidate residual layouts for the single-RHS kernel:
row predictor order (1, 2, 3), optional column difference inside the chunk,
chunk length, at byte granularity of the chunk width (and the bit floor).

usage: python tools/predictor_study.py CFG [ROW_STEP]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import configs

cfg = configs.get(int(sys.argv[1]))
step = int(sys.argv[2]) if len(sys.argv) > 2 else 8
N = cfg.N
grid = 148
dop = invop.DeviceOperator(cfg.operator()).factor()


def widths(e, CH):
    nch = (N + CH - 1) // CH
    pad = torch.nn.functional.pad(e.abs(), (0, nch * CH - N))
    mx = pad.view(e.shape[0], nch, CH).amax(dim=2).double()
    return torch.ceil(torch.log2(mx + 1)) + 1          # signed bits


acc = {}
for b in range(0, grid, step):
    lo, hi = b * N // grid, (b + 1) * N // grid
    m = dop.quantized_rows(cfg.digits, lo, hi - lo).decode().long()
    d1 = m[1:] - m[:-1]
    d2 = d1[1:] - d1[:-1]
    d3 = d2[1:] - d2[:-1]
    for name, e in (("row1", d1[2:]), ("row2", d2[1:]), ("row3", d3)):
        for col in (0, 1):
            for CH in (512, 256, 128, 64):
                ee = e
                if col:
                    # column difference restarting at every chunk
                    ee = e.clone()
                    ee[:, 1:] -= e[:, :-1]
                    ee[:, ::CH] = e[:, ::CH]
                bt = widths(ee, CH)
                key = (name, col, CH)
                a = acc.setdefault(key, [0.0, 0.0, 0])
                a[0] += float(torch.ceil(bt / 8).clamp(min=1).sum())
                a[1] += float((bt / 8).sum())
                a[2] += bt.numel()
print("config", cfg.key, "rows sampled every", step, "CTA ranges")
for (name, col, CH), (by, bi, n) in sorted(acc.items()):
    print("%s %s chunk %3d: byte-granular %.3f B/entry (+%.3f header at 1 B/chunk), bit floor %.3f" % (
        name, "+coldiff" if col else "        ", CH, by / n, 1.0 / CH, bi / n))
