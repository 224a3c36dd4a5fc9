"""Time the ordered (bitwise fp64) apply of a config on the resident operator.

usage: python tools/time_ordered.py CONFIG [NRHS] [REPS]
Prints ms per apply and GB/s on the byte planes the kernel streams.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C
import os

import numpy as np
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import _lib as L, configs

key = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = configs.get(key)
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 100
st = cfg.operator()
plan = invop.DeviceOperator(st).factor().quantized_rows(cfg.digits)
N = st.n
R = np.asarray(cfg.rhs())
R = np.tile(R, (-(-k // R.shape[0]), 1))[:k]
x = torch.tensor(R, device="cuda").contiguous()
y64 = torch.empty(k, N, device="cuda", dtype=torch.float64)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
h = plan.handle


def run():
    L.check(L.lib.invop_apply(h, x.data_ptr(), N, y64.data_ptr(), N, k, L.F64, L.MODE_ORDERED, s))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
ob = C.c_int64(0)
L.check(L.lib.invop_plan_apply_bytes(h, k, L.MODE_ORDERED, C.byref(ob), s))
env = " ".join("%s=%s" % kv for kv in sorted(os.environ.items()) if kv[0].startswith("INVOP_"))
print("ordered cfg %d k=%d [%s]: %.4f ms/apply  %.0f GB/s on %.1f MB  sum %.17g" % (
    key, k, env, ms, ob.value / ms / 1e6, ob.value / 1e6, float(y64.sum())), flush=True)
