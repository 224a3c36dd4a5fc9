"""Row-delta statistics of a config's quantized operator: bytes needed by
d_r = v_r - v_{r-1} per 512-column chunk (and per K3 128x64 tile). Needs a GPU.

usage: python tools/delta_stats.py CFG [ROWS_PER_BLOCK] [d1|d2|dnx]
  d1: d_r = v_r - v_{r-1};  d2: v_r - 2 v_{r-1} + v_{r-2};  dnx: v_r - v_{r-nx}
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import configs

cfg = configs.get(int(sys.argv[1]))
rb = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
mode = sys.argv[3] if len(sys.argv) > 3 else "d1"
CH = int(sys.argv[4]) if len(sys.argv) > 4 else 512
dop = invop.DeviceOperator(cfg.operator()).factor()
N = cfg.N
nch = (N + CH - 1) // CH
hist = torch.zeros(5, dtype=torch.int64, device="cuda")     # chunks needing 1..4 bytes (index 0 unused)
ehist = torch.zeros(5, dtype=torch.int64, device="cuda")    # entries needing 1..4 bytes
thist = torch.zeros(5, dtype=torch.int64, device="cuda")    # K3 tiles needing 1..4 bytes
prev = None


def width(a):
    w = torch.ones_like(a, dtype=torch.int64)
    w = torch.where(a > 127, 2, w)
    w = torch.where(a > 32767, 3, w)
    w = torch.where(a > 8388607, 4, w)
    return w


for r0 in range(0, N, rb):
    rows = min(rb, N - r0)
    back = {"d1": 1, "d2": 2, "dnx": cfg.n, "p2d": cfg.n + 1, "d2nx": 2 * cfg.n}[mode]
    lo = max(r0 - back, 0)
    m = dop.quantized_rows(cfg.digits, lo, rows + (r0 - lo)).decode()
    if r0 - lo < back:   # first block: zero rows before row 0
        m = torch.cat([torch.zeros((back - (r0 - lo), N), dtype=m.dtype, device=m.device), m])
    if mode == "d2":
        d = m[2:] - 2 * m[1:-1] + m[:-2]
    elif mode == "p2d":     # v_r - v_{r-1} - v_{r-nx} + v_{r-nx-1}
        nx = cfg.n
        d = m[back:] - m[back - 1:-1] - m[1:-(nx)] + m[:-(nx + 1)]
    elif mode == "d2nx":    # second difference across grid lines
        nx = cfg.n
        d = m[2 * nx:] - 2 * m[nx:-nx] + m[:-2 * nx]
    else:
        d = m[back:] - m[:-back]
    a = d.abs()
    pad = torch.nn.functional.pad(a, (0, nch * CH - N))
    cw = width(pad.view(rows, nch, CH).amax(dim=2))
    hist += torch.bincount(cw.flatten(), minlength=5)
    ehist += torch.bincount(width(a).flatten(), minlength=5)
    if rows % 128 == 0:
        nk = (N + 63) // 64
        pad = torch.nn.functional.pad(a, (0, nk * 64 - N))
        tw = width(pad.view(rows // 128, 128, nk, 64).amax(dim=(1, 3)))
        thist += torch.bincount(tw.flatten(), minlength=5)
    del m, d, a, pad
h = hist.cpu().tolist()
e = ehist.cpu().tolist()
t = thist.cpu().tolist()
tot = sum(h)
print("config", cfg.key, "N", N, "mode", mode, "chunk", CH)
print("chunks by delta width (1..4 B):", [round(x / tot, 4) for x in h[1:]],
      "-> B/entry %.3f" % (sum(w * h[w] for w in range(1, 5)) / tot))
print("entries by delta width:", [round(x / sum(e), 4) for x in e[1:]])
if sum(t):
    print("K3 tiles by delta width:", [round(x / sum(t), 4) for x in t[1:]],
          "-> planes/tile %.3f" % (sum(w * t[w] for w in range(1, 5)) / sum(t)))
