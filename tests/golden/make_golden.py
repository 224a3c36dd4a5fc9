"""Generate the golden fixtures of tests/golden/ by importing the REFERENCE
package itself (/root/reference/pkg/src, read-only; pure-Python backend,
which the reference guarantees bitwise equal to its compiled one,
_kernels/_native.pyx:4-10).

Run in the build container only (the GPU box has no /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
The fixtures are small .npz files; tests read them, never this script.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))
import invop  # noqa: E402  (the reference)

OUT = Path(__file__).resolve().parent


def random_quantized(rng, n, digits):
    """Same generator as the reference's tests/conftest.py:33-38."""
    pool = rng.integers(1, 10 ** (digits + 1) + 9, size=int(rng.integers(1, 5)))
    mant = rng.choice(pool, size=(n, n)) * rng.choice([-1, 0, 1], size=(n, n))
    return invop.QuantizedMatrix(n=n, scale_digits=digits, mantissas=mant.astype(np.int64))


def battery(seed, trials):
    """Reference test_oracle_equality_random_battery (seed 2024, 60 trials) and
    acceptance criterion 3 (seed 7, 220 trials)."""
    rng = np.random.default_rng(seed)
    mants, xs, ys, yn, meta = [], [], [], [], []
    for _ in range(trials):
        n = int(rng.integers(2, 17))
        m = int(rng.integers(0, 5))
        q = random_quantized(rng, n, m)
        x = rng.standard_normal(n)
        plan = invop.build_plan(q)
        y, c = invop.apply(plan, x)
        y2, c2 = invop.apply_naive_quantized(q, x)
        assert y.tobytes() == y2.tobytes()
        mants.append(q.mantissas.ravel()); xs.append(x); ys.append(y)
        meta.append((n, m, c.multiplications, c.additions))
    meta = np.array(meta, dtype=np.int64)
    return dict(meta=meta, mant=np.concatenate(mants), x=np.concatenate(xs), y=np.concatenate(ys))


def plan_tables(q):
    p = invop.build_plan(q)
    return {k: getattr(p, k) for k in ("col_ptr", "group_abs_mantissa", "group_coeff",
                                       "group_ptr", "entry_rows", "entry_signs")}


def grid_cases():
    out = {}
    for side in (5, 11):
        grid = invop.Grid2D(side, side)
        op = invop.build_uniform(grid)
        ainv = invop.invert(op)
        rhs = invop.assemble_rhs(grid, invop.SourceField(f=invop.test_source))
        out["g%d_inverse" % side] = ainv.entries
        out["g%d_rhs" % side] = rhs
        ud, cd = invop.apply_dense(ainv, rhs)
        out["g%d_dense_y" % side] = ud
        for m in (1, 2, 3, 5):
            q = invop.quantize(ainv, m)
            plan = invop.build_plan(q)
            y, c = invop.apply(plan, rhs)
            nz, distinct = invop.sparsity_stats(q)
            out["g%d_m%d_mant" % (side, m)] = q.mantissas
            out["g%d_m%d_y" % (side, m)] = y
            out["g%d_m%d_counts" % (side, m)] = np.array([c.multiplications, c.additions])
            out["g%d_m%d_distinct" % (side, m)] = np.array(distinct)
            out["g%d_m%d_relerr" % (side, m)] = np.array([invop.relative_error(y, grid)])
            if side == 5:
                for k, v in plan_tables(q).items():
                    out["g5_m%d_%s" % (m, k)] = v
    # 3x5 grid (reference test_quant / test_applyplan use it)
    g35 = invop.Grid2D(3, 5)
    a35 = invop.invert(invop.build_uniform(g35))
    out["g35_inverse"] = a35.entries
    out["g35_m0_mant"] = invop.quantize(a35, 0).mantissas
    # variable-coefficient full-grid operator
    g = invop.Grid2D(6, 5)
    beta = np.linspace(0.5, 1.5, g.n)
    opv = invop.build_variable(g, invop.CoefficientField(beta))
    out["var_entries"] = opv.entries
    out["var_beta"] = beta
    out["var_inverse"] = invop.invert(opv).entries
    return out


def interior_uniform_dense(n):
    N = n * n
    a = np.eye(N)
    for p in range(N):
        r, c = divmod(p, n)
        for rr, cc in ((r, c - 1), (r, c + 1), (r - 1, c), (r + 1, c)):
            if 0 <= rr < n and 0 <= cc < n:
                a[p, rr * n + cc] = -0.25
    return a


def config1():
    """BASELINE config 1: uniform 10x10 interior, m=3, rho ~ rng(101) N(0,1), fp64."""
    a = interior_uniform_dense(10)
    ainv = invop.invert(invop.DenseMatrix(n=100, entries=a))
    q = invop.quantize(ainv, 3)
    x = np.random.default_rng(101).standard_normal(100)
    y, c = invop.apply(invop.build_plan(q), x)
    return dict(inverse=ainv.entries, mant=q.mantissas, x=x, y=y,
                counts=np.array([c.multiplications, c.additions]))


def config2():
    """BASELINE config 2: uniform 50x50 interior, m=4, 16 RHS rng(102); the
    full mantissa matrix (12.5 MB as int16) is summarised, outputs are kept."""
    a = interior_uniform_dense(50)
    ainv = invop.invert(invop.DenseMatrix(n=2500, entries=a))
    q = invop.quantize(ainv, 4)
    X = np.random.default_rng(102).standard_normal((16, 2500))
    plan = invop.build_plan(q)
    Y = np.stack([invop.apply(plan, X[t])[0] for t in range(16)])
    mant = q.mantissas
    nz, distinct = invop.sparsity_stats(q)
    return dict(X=X, Y=Y, mant_sum=np.array([mant.sum()]), mant_sq=np.array([(mant.astype(np.float64) ** 2).sum()]),
                mant_max=np.array([mant.max()]), distinct=np.array(distinct), nnz=np.array([nz]),
                counts=np.array([plan.planned_multiplications, plan.planned_additions]),
                rows_sample=np.array([0, 1, 1234, 1275, 2499]), mant_rows=mant[[0, 1, 1234, 1275, 2499]])


def quant_cases():
    vals = np.array([0.12345, -0.005, 0.005, 0.025, -0.35, 0.5, -0.5, 1.5, 2.5, 1e-7, 123.456789])
    out = {"vals": vals}
    for m in range(0, 7):
        out["m%d" % m] = np.array([invop.quantize(invop.DenseMatrix(n=1, entries=np.array([[v]])), m).mantissas[0, 0]
                                   for v in vals])
    rng = np.random.default_rng(5)
    mat = rng.uniform(-1, 1, (8, 8))
    out["rand8"] = mat
    for m in (0, 3, 6, 12):
        out["rand8_m%d" % m] = invop.quantize(invop.DenseMatrix(n=8, entries=mat), m).mantissas
    return out


def main():
    np.savez_compressed(OUT / "battery_2024.npz", **battery(2024, 60))
    np.savez_compressed(OUT / "battery_7.npz", **battery(7, 220))
    np.savez_compressed(OUT / "grid_cases.npz", **grid_cases())
    np.savez_compressed(OUT / "config1.npz", **config1())
    np.savez_compressed(OUT / "quant_cases.npz", **quant_cases())
    np.savez_compressed(OUT / "config2.npz", **config2())
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
