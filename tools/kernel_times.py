"""Live per-kernel device times of a config's apply (CUPTI via torch.profiler;
no replay, no cache flush — unlike the ncu launch list).

usage: python tools/kernel_times.py CONFIG [fast|ordered] [NRHS] [ITERS]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C
from collections import defaultdict

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import _lib as L, configs

cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 1
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20
st = cfg.operator()
plan = invop.DeviceOperator(st).factor().quantized_rows(cfg.digits)
N = st.n
R = np.asarray(cfg.rhs())
R = np.tile(R, (-(-k // R.shape[0]), 1))[:k]
x64 = torch.tensor(R, device="cuda").contiguous()
x32 = x64.float()
y32 = torch.empty(k, N, device="cuda")
y64 = torch.empty(k, N, device="cuda", dtype=torch.float64)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def run():
    if mode == "fast":
        L.check(L.lib.invop_apply(plan.handle, x32.data_ptr(), N, y32.data_ptr(), N, k, L.F32, L.MODE_FAST, s))
    else:
        L.check(L.lib.invop_apply(plan.handle, x64.data_ptr(), N, y64.data_ptr(), N, k, L.F64, L.MODE_ORDERED, s))


for _ in range(3):
    run()
torch.cuda.synchronize()
st_ev, en_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st_ev.record()
for _ in range(iters):
    run()
en_ev.record()
torch.cuda.synchronize()
wall = st_ev.elapsed_time(en_ev) / iters * 1e3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(iters):
        run()
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type.name == "CUDA" or getattr(ev, "device_time", 0):
        dt = getattr(ev, "device_time", None) or getattr(ev, "cuda_time", 0)
        if dt:
            agg[ev.name][0] += 1
            agg[ev.name][1] += dt
print("config %d mode %s nrhs %d: %.1f us per apply (events, back to back)" % (cfg.key, mode, k, wall))
tot = 0.0
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    tot += t / iters
    print("%5d x %9.1f us  (%8.1f us/apply)  %s" % (n, t / n, t / iters, name[:100]))
print("sum of kernel times per apply: %.1f us" % tot)
