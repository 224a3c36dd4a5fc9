"""Time the fast single-RHS apply of a row shard of a config (what one rank of
an N-GPU run executes): python tools/time_shard.py CONFIG WORLD [REPS]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C
import os

import numpy as np
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import _lib as L, configs
from paper_1602_00001_b200.sharded import shard_rows

cfg = configs.get(int(sys.argv[1]))
world = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
k = int(sys.argv[4]) if len(sys.argv) > 4 else 1
st = cfg.operator()
N = st.n
row0, rows = shard_rows(N, world, 0)
plan = invop.DeviceOperator(st).factor().quantized_rows(cfg.digits, row0, rows)
R = np.asarray(cfg.rhs())
R = np.tile(R, (-(-k // R.shape[0]), 1))[:k]
x32 = torch.tensor(R, device="cuda", dtype=torch.float32).contiguous()
y32 = torch.empty(k, rows, device="cuda")
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
h = plan.handle


def run():
    L.check(L.lib.invop_apply(h, x32.data_ptr(), N, y32.data_ptr(), rows, k, L.F32, L.MODE_FAST, s))


for _ in range(5):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
# isolated: a synchronisation after every apply
ts = []
for _ in range(50):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ob = C.c_int64(0)
L.check(L.lib.invop_plan_apply_bytes(h, k, L.MODE_FAST, C.byref(ob), s))
env = " ".join("%s=%s" % kv for kv in sorted(os.environ.items()) if kv[0].startswith("INVOP_") and kv[0] != "INVOP_B200_LIB")
print("cfg %d shard 1/%d (%d rows) k=%d [%s] %s: %.4f ms back to back, %.4f ms isolated, %.0f GB/s on %.1f MB" % (
    cfg.key, world, rows, k, env, L.lib.invop_apply_kernel(h, k, L.MODE_FAST).decode(), ms,
    float(np.median(ts)), ob.value / ms / 1e6, ob.value / 1e6), flush=True)
