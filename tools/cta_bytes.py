"""Bytes per CTA of the DL layout (byte widths per 512-column chunk), i.e. the
load balance of k2_dl across the 148 CTAs (equal row counts per CTA).

usage: python tools/cta_bytes.py CFG
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import configs

cfg = configs.get(int(sys.argv[1]))
N = cfg.N
grid = 148
dop = invop.DeviceOperator(cfg.operator()).factor()
CH = 512
nch = (N + CH - 1) // CH


def bwidth(e):
    w = torch.ones_like(e, dtype=torch.int64)
    for b in range(1, 4):
        lim = 128 * 256 ** (b - 1)
        w = torch.where((e >= lim) | (e < -lim), b + 1, w)
    return w


per = []
for b in range(grid):
    lo, hi = b * N // grid, (b + 1) * N // grid
    m = dop.quantized_rows(cfg.digits, lo, hi - lo).decode()
    e = m.clone()
    e[1:] -= m[:-1]
    e[2:] -= m[1:-1] - m[:-2]
    pad = torch.nn.functional.pad(e, (0, nch * CH - N))
    W = bwidth(pad.view(hi - lo, nch, CH)).amax(dim=2)
    per.append(float(W.sum()) * 512 + 48 * (hi - lo))
t = torch.tensor(per)
print("config", int(sys.argv[1]), "bytes per CTA: mean %.2f MB  max %.2f MB  min %.2f MB  max/mean %.3f" % (
    t.mean() / 1e6, t.max() / 1e6, t.min() / 1e6, float(t.max() / t.mean())))
print("deciles:", [round(float(x) / 1e6, 2) for x in torch.quantile(t, torch.linspace(0, 1, 11))])
