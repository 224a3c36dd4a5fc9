"""K3 probe: random 2-byte codes rows x n, 64 RHS (for timing / ncu)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_1602_00001_b200 as invop

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = torch.Generator(device="cuda").manual_seed(0)
mant = torch.randint(0, 40000, (rows, n), device="cuda", dtype=torch.int64, generator=g)
dplan = invop._plan.DevicePlan.from_mantissas(mant, 4, row0=0, n=n)
del mant
X = torch.randn(64, n, device="cuda", generator=g)
Y = dplan.apply_device(X, mode=0)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(reps):
    Y = dplan.apply_device(X, mode=0)
t1.record(); torch.cuda.synchronize()
ms = t0.elapsed_time(t1) / reps
print("rows=%d n=%d: %.3f ms per 64-RHS apply, %.1f GB/s codes" % (rows, n, ms, rows * n * 2 / ms / 1e6))
