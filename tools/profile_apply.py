"""Run a config's apply kernels a few times (for ncu captures).

usage: python tools/profile_apply.py CONFIG [fast,ordered] [NRHS]
NRHS > 1 runs the batched (K3) path on the config's first NRHS right-hand sides.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C

import numpy as np
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import _lib as L, configs

cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fast", "ordered"]
k = int(sys.argv[3]) if len(sys.argv) > 3 else 1
st = cfg.operator()
plan = invop.DeviceOperator(st).factor().quantized_rows(cfg.digits)
N = st.n
R = np.asarray(cfg.rhs())
R = np.tile(R, (-(-k // R.shape[0]), 1))[:k]
x = torch.tensor(R, device="cuda").contiguous()
x32 = x.float()
y32 = torch.empty(k, N, device="cuda")
y64 = torch.empty(k, N, device="cuda", dtype=torch.float64)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    if "fast" in modes:
        L.check(L.lib.invop_apply(plan.handle, x32.data_ptr(), N, y32.data_ptr(), N, k, L.F32, L.MODE_FAST, s))
    if "ordered" in modes:
        L.check(L.lib.invop_apply(plan.handle, x.data_ptr(), N, y64.data_ptr(), N, k, L.F64, L.MODE_ORDERED, s))
torch.cuda.synchronize()
print("ok", plan.code_bytes)
