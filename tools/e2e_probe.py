"""Break the end-to-end host apply of a config into its parts (per call, us).

usage: python tools/e2e_probe.py CONFIG [CALLS]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C

import numpy as np
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import _lib as L, configs

key = int(sys.argv[1]) if len(sys.argv) > 1 else 4
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
cfg = configs.get(key)
st = cfg.operator()
plan = invop.DeviceOperator(st).factor().quantized_rows(cfg.digits)
N = st.n
h = plan.handle
stream = torch.cuda.current_stream()
s = C.c_void_p(stream.cuda_stream)
xh = torch.from_numpy(np.asarray(cfg.rhs())[0].copy()).pin_memory()
yh = torch.empty(N, dtype=torch.float64).pin_memory()
xd = torch.empty(N, dtype=torch.float64, device="cuda")
x32 = torch.empty(N, device="cuda")
y32 = torch.empty(N, device="cuda")
xp, yp = xh.data_ptr(), yh.data_ptr()
f = L.lib.invop_apply_host


def per_call(fn, n=calls):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def full():
    f(h, xp, yp, 1, L.MODE_FAST, s)


def sync_only():
    torch.cuda.synchronize()


def h2d_sync():
    xd.copy_(xh, non_blocking=True)
    torch.cuda.synchronize()


def kernel_sync():
    L.lib.invop_apply(h, x32.data_ptr(), N, y32.data_ptr(), N, 1, L.F32, L.MODE_FAST, s)
    torch.cuda.synchronize()


def kernel_only():
    L.lib.invop_apply(h, x32.data_ptr(), N, y32.data_ptr(), N, 1, L.F32, L.MODE_FAST, s)


def ctypes_nop():
    L.lib.invop_last_error()


for name, fn in [("ctypes call", ctypes_nop), ("synchronize", sync_only), ("H2D 128KB + sync", h2d_sync),
                 ("kernel back-to-back", kernel_only), ("kernel + sync", kernel_sync),
                 ("invop_apply_host", full)]:
    print("%-22s %8.2f us" % (name, per_call(fn)), flush=True)
