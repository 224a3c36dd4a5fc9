"""Grouped (reference-shaped) apply vs the exact-integer kernels at config 4.

DESIGN.md "No grouping on the device": times invop_apply_grouped_csc (the
reference's CSC group loop, _native.pyx:15-49, on device tables built by
invop_plan_csc) against the default fp32 route (k2_dl) and the bitwise fp64
route (k2_ordered) on the same plan and x, and prints one JSON line with the
bytes each streams. Run the ncu launch list of this script for DRAM bytes.

usage: python tools/grouped_baseline.py [CONFIG]
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import _lib as L, configs

cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
st = cfg.operator()
plan = invop.DeviceOperator(st).factor().quantized_rows(cfg.digits)
N = st.n
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
G, E = C.c_int64(), C.c_int64()
L.check(L.lib.invop_plan_csc(plan.handle, None, None, None, None, None, None, C.byref(G), C.byref(E), s))
g, e = G.value, E.value
col_ptr = torch.zeros(N + 1, dtype=torch.int64, device="cuda")
gabs = torch.empty(g, dtype=torch.int64, device="cuda")
gcoeff = torch.empty(g, dtype=torch.float64, device="cuda")
gptr = torch.zeros(g + 1, dtype=torch.int64, device="cuda")
rows = torch.empty(e, dtype=torch.int32, device="cuda")
signs = torch.empty(e, dtype=torch.int8, device="cuda")
L.check(L.lib.invop_plan_csc(plan.handle, col_ptr.data_ptr(), gabs.data_ptr(), gcoeff.data_ptr(),
                             gptr.data_ptr(), rows.data_ptr(), signs.data_ptr(), C.byref(G), C.byref(E), s))
del gabs
x64 = torch.tensor(cfg.rhs()[0], device="cuda", dtype=torch.float64)
x32 = x64.float()
yg = torch.empty(N, device="cuda", dtype=torch.float64)
y64 = torch.empty(N, device="cuda", dtype=torch.float64)
y32 = torch.empty(N, device="cuda", dtype=torch.float32)


def grouped():
    L.check(L.lib.invop_apply_grouped_csc(N, col_ptr.data_ptr(), gcoeff.data_ptr(), gptr.data_ptr(),
                                          rows.data_ptr(), signs.data_ptr(), x64.data_ptr(),
                                          yg.data_ptr(), s))


def fast():
    L.check(L.lib.invop_apply(plan.handle, x32.data_ptr(), N, y32.data_ptr(), N, 1, L.F32, L.MODE_FAST, s))


def ordered():
    L.check(L.lib.invop_apply(plan.handle, x64.data_ptr(), N, y64.data_ptr(), N, 1, L.F64,
                              L.MODE_ORDERED, s))


def time_ms(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


tg, tf, to = time_ms(grouped, 20), time_ms(fast, 200), time_ms(ordered, 50)
ob = C.c_int64()
L.check(L.lib.invop_plan_apply_bytes(plan.handle, 1, L.MODE_FAST, C.byref(ob), s))
ordb = C.c_int64()
L.check(L.lib.invop_plan_apply_bytes(plan.handle, 1, L.MODE_ORDERED, C.byref(ordb), s))
rel = float(((yg - y64).abs().max() / y64.abs().max()).item())
grouped_bytes = 16 * g + 5 * e + 8 * (N + 1)
print(json.dumps({
    "config": cfg.key, "N": N, "groups": g, "entries": e,
    "grouped_csc": {"ms": tg, "table_bytes": grouped_bytes, "gbs": grouped_bytes / tg / 1e6,
                    "relerr_vs_ordered": rel, "note": "reference loop on device tables, fp64 atomics"},
    "k2_dl_fp32": {"ms": tf, "operator_bytes": ob.value, "gbs": ob.value / tf / 1e6},
    "ordered_fp64": {"kernel": L.lib.invop_apply_kernel(plan.handle, 1, L.MODE_ORDERED).decode(),
                     "ms": to, "operator_bytes": ordb.value, "gbs": ordb.value / to / 1e6},
    "speedup_exact_over_grouped": tg / tf,
}))
