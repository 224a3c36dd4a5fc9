"""Residual magnitude per (row, 512-column chunk) of the DL layout: bytes per
entry at byte, nibble and bit granularity of the chunk width.

usage: python tools/width_hist.py CFG [ROW_STEP]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import configs

cfg = configs.get(int(sys.argv[1]))
step = int(sys.argv[2]) if len(sys.argv) > 2 else 1
N = cfg.N
grid = 148
dop = invop.DeviceOperator(cfg.operator()).factor()
CH = 512
nch = (N + CH - 1) // CH
bits = []
for b in range(0, grid, step):
    lo, hi = b * N // grid, (b + 1) * N // grid
    m = dop.quantized_rows(cfg.digits, lo, hi - lo).decode()
    e = m.clone()
    e[1:] -= m[:-1]
    e[2:] -= m[1:-1] - m[:-2]
    e = e[2:]                                   # order-2 rows only
    pad = torch.nn.functional.pad(e.abs(), (0, nch * CH - N))
    mx = pad.view(e.shape[0], nch, CH).amax(dim=2).double()
    # signed width in bits: smallest w with -2^(w-1) <= e < 2^(w-1)
    bits.append(torch.ceil(torch.log2(mx + 1)) + 1)
bt = torch.cat([x.flatten() for x in bits])
byte = torch.ceil(bt / 8).clamp(min=1)
nib = torch.ceil(bt / 4).clamp(min=1) / 2
print("config", int(sys.argv[1]), "chunks", bt.numel())
print("B/entry: byte %.3f  nibble %.3f  bit %.3f" % (byte.mean(), nib.mean(), (bt / 8).mean()))
h = torch.bincount(bt.long(), minlength=26)[:26].tolist()
print("chunk signed-bit histogram:", {i: round(v / bt.numel(), 4) for i, v in enumerate(h) if v})
