"""Per-consumer-warp work balance of the DL layout (k2_dl): residual planes per
warp (chunks c and c+16 of every 16384-column slab) summed over each CTA's rows.

usage: python tools/dl_balance.py CFG
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
        lim = 128 * 256 ** (b - 1)     # balanced: |e| < 128*256^(b-1) roughly
        w = torch.where((e >= lim) | (e < -lim), b + 1, w)
    return w


W = torch.zeros(N, nch, dtype=torch.int64, device="cuda")
for b in range(grid):
    lo, hi = b * N // grid, (b + 1) * N // grid
    m = dop.quantized_rows(cfg.digits, lo, hi - lo).decode()
    e = m.clone()
    e[1:] -= m[:-1]
    e[2:] -= m[1:-1] - m[:-2]
    pad = torch.nn.functional.pad(e, (0, nch * CH - N))
    W[lo:hi] = bwidth(pad.view(hi - lo, nch, CH)).amax(dim=2)
nsl = (nch + 31) // 32
ratios, hot = [], []
warp_cost = torch.zeros(grid, 16, device="cuda")
for b in range(grid):
    lo, hi = b * N // grid, (b + 1) * N // grid
    Wb = W[lo:hi].float()
    Wb = torch.nn.functional.pad(Wb, (0, nsl * 32 - nch))
    per = Wb.view(hi - lo, nsl, 2, 16).sum(dim=(0, 1, 2))     # per warp: chunks wc, wc+16 over slabs
    warp_cost[b] = per
    ratios.append(float(per.max() / per.mean()))
r = torch.tensor(ratios)
print("config", int(sys.argv[1]), "mean planes per chunk %.3f" % float(W.float().mean()))
print("per-CTA max/mean warp planes: mean %.3f  max %.3f  min %.3f" % (r.mean(), r.max(), r.min()))
# with ~100 instructions of per-row overhead per warp and 12 DP4A per plane
rows = N / grid
fixed = 100 * nsl * rows
c = 12 * warp_cost + fixed
print("est. issue-time ratio max/mean (100 instr/row overhead): %.3f" % float((c.max(1).values / c.mean(1)).mean()))
print("width histogram:", torch.bincount(W.flatten(), minlength=5).tolist())
