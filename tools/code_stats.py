"""Byte-width statistics of a config's quantized operator (which chunks/tiles
need which code bytes), for layout decisions. Needs a GPU.

usage: python tools/code_stats.py CFG [ROWS_PER_BLOCK]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import configs

cfg = configs.get(int(sys.argv[1]))
rb = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
dop = invop.DeviceOperator(cfg.operator()).factor()
N = cfg.N
tot = {}
def add(k, v):
    tot[k] = tot.get(k, 0) + v
for r0 in range(0, N, rb):
    rows = min(rb, N - r0)
    pl = dop.quantized_rows(cfg.digits, r0, rows)
    m = pl.decode()                                   # [rows, N] int64
    a = m.abs()
    add("entries", m.numel())
    add("zero", int((m == 0).sum()))
    for b, lim in ((1, 127), (2, 32767), (3, 8388607)):
        add("abs>%d" % lim, int((a > lim).sum()))
    # 512-column chunks along a row
    nch = (N + 511) // 512
    pad = torch.nn.functional.pad(a, (0, nch * 512 - N))
    cm = pad.view(rows, nch, 512).amax(dim=2)
    add("chunks", cm.numel())
    for lim in (0, 127, 32767):
        add("chunk max>%d" % lim, int((cm > lim).sum()))
    # K3 tiles: 128 rows x 64 columns
    if rows % 128 == 0:
        nk = (N + 63) // 64
        pad = torch.nn.functional.pad(a, (0, nk * 64 - N))
        tm = pad.view(rows // 128, 128, nk, 64).amax(dim=(1, 3))
        add("tiles", tm.numel())
        for lim in (0, 127, 255, 32767):
            add("tile max>%d" % lim, int((tm > lim).sum()))
    del m, a, pad
print("config", cfg.key, "N", N, "digits", cfg.digits, "max", float(dop.quantized_rows(cfg.digits, 0, 1).decode().abs().max()))
for k, v in tot.items():
    base = tot["entries"] if k in ("zero",) or k.startswith("abs") else (
        tot["chunks"] if k.startswith("chunk") else tot.get("tiles", 1))
    print("%-18s %14d  %.4f" % (k, v, v / base))
