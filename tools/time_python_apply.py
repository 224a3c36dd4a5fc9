"""Wall time of the Python drop-in call with numpy arrays (pageable host
memory): invop.apply(plan, x) in both precisions.
usage: python tools/time_python_apply.py CONFIG [REPS]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import os

import numpy as np
import torch

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import configs

cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
st = cfg.operator()
dplan = invop.DeviceOperator(st).factor().quantized_rows(cfg.digits)
plan = invop.ApplyPlan(n=st.n, scale_digits=cfg.digits, _dplan=dplan)
x = np.asarray(cfg.rhs())[0].astype(np.float64)
env = " ".join("%s=%s" % kv for kv in sorted(os.environ.items()) if kv[0].startswith("INVOP_") and kv[0] != "INVOP_B200_LIB")
for prec in ("f64", "f32"):
    for _ in range(5):
        y, _ = invop.apply(plan, x, precision=prec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        y, _ = invop.apply(plan, x, precision=prec)
    dt = (time.perf_counter() - t0) / reps
    print("cfg %d invop.apply(plan, numpy x, precision=%s) [%s]: %.1f us per call, %.0f applies/s" % (
        cfg.key, prec, env, dt * 1e6, 1.0 / dt), flush=True)
