"""Bitwise parity of the b200 backend with the reference's own backends.

Staged into the reference package's tests/ by integration/stage_reference.py
and run there (tests/test_reference_suite.py, on a GPU). The pattern is the
reference's compiled-vs-Python parity suite (pkg/tests/test_backends.py:25-87):
the same kernel signature called on the same tables, outputs compared byte
for byte and operation counts compared exactly — here the device backend
(`invop._kernels._b200`, libinvop_b200.so) against `_native` (the
reference's compiled kernel) and `_fallback` (its Python twin).
"""

import numpy as np
import pytest

import invop
from invop._kernels import _fallback
from conftest import random_quantized

_b200 = pytest.importorskip("invop._kernels._b200")
try:
    from invop._kernels import _native
except ImportError:          # the staged copy ships without a compiled kernel
    _native = None

_REFS = [("python", _fallback)] + ([("native", _native)] if _native is not None else [])


def _plan_inputs(seed, n=12, m=3):
    rng = np.random.default_rng(seed)
    q = random_quantized(rng, n, m)
    plan = invop.build_plan(q)
    x = rng.standard_normal(n)
    return plan, q, x


def test_backend_is_b200():
    assert invop.BACKEND == "b200"


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("n,m", [(12, 3), (1, 0), (40, 5), (129, 6)])
def test_plan_apply_parity(seed, n, m):
    plan, _, x = _plan_inputs(seed, n, m)
    args = (plan.col_ptr, plan.group_coeff, plan.group_ptr, plan.entry_rows, plan.entry_signs)
    out_d = np.zeros(plan.n)
    counts_d = _b200.plan_apply(*args, x, out_d)
    for name, ref in _REFS:
        out_r = np.zeros(plan.n)
        counts_r = ref.plan_apply(*args, x, out_r)
        assert tuple(counts_d) == tuple(counts_r), name
        assert out_d.tobytes() == out_r.tobytes(), name


@pytest.mark.parametrize("seed", range(4))
def test_plan_apply_accumulates_into_out(seed):
    """The kernel adds into the caller's buffer (_native.pyx:43-46)."""
    plan, _, x = _plan_inputs(seed, 17, 2)
    args = (plan.col_ptr, plan.group_coeff, plan.group_ptr, plan.entry_rows, plan.entry_signs)
    start = np.random.default_rng(seed + 50).standard_normal(plan.n)
    out_d, out_r = start.copy(), start.copy()
    _b200.plan_apply(*args, x, out_d)
    _fallback.plan_apply(*args, x, out_r)
    assert out_d.tobytes() == out_r.tobytes()


def test_plan_apply_nonfinite_x():
    """inf/nan in x: zero mantissas are skipped, as in the reference loop."""
    plan, _, x = _plan_inputs(3, 12, 3)
    x = x.copy()
    x[2], x[5] = np.inf, np.nan
    args = (plan.col_ptr, plan.group_coeff, plan.group_ptr, plan.entry_rows, plan.entry_signs)
    out_d, out_r = np.zeros(plan.n), np.zeros(plan.n)
    _b200.plan_apply(*args, x, out_d)
    _fallback.plan_apply(*args, x, out_r)
    assert out_d.tobytes() == out_r.tobytes()


@pytest.mark.parametrize("seed", range(8))
def test_naive_apply_parity(seed):
    _, q, x = _plan_inputs(seed, n=9, m=2)
    mant_t = q.mantissas.T
    cols, rows = np.nonzero(mant_t)
    vals = mant_t[cols, rows].astype(np.float64) * q.scale
    col_ptr = np.zeros(q.n + 1, dtype=np.int64)
    col_ptr[1:] = np.cumsum(np.bincount(cols, minlength=q.n))
    rows32 = rows.astype(np.int32)
    out_d = np.zeros(q.n)
    counts_d = _b200.naive_apply(col_ptr, rows32, vals, x, out_d)
    for name, ref in _REFS:
        out_r = np.zeros(q.n)
        counts_r = ref.naive_apply(col_ptr, rows32, vals, x, out_r)
        assert tuple(counts_d) == tuple(counts_r), name
        assert out_d.tobytes() == out_r.tobytes(), name


@pytest.mark.parametrize("seed", range(4))
def test_dense_matvec_parity(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 30))
    mat = np.ascontiguousarray(rng.standard_normal((n, n)))
    x = rng.standard_normal(n)
    out_d = np.zeros(n)
    counts_d = _b200.dense_matvec(mat, x, out_d)
    for name, ref in _REFS:
        out_r = np.zeros(n)
        counts_r = ref.dense_matvec(mat, x, out_r)
        assert tuple(counts_d) == tuple(counts_r) == (n * n, n * (n - 1)), name
        assert out_d.tobytes() == out_r.tobytes(), name


def test_grid_pipeline_matches_python_backend(cells):
    """Whole reference pipeline on a grid inverse (build_uniform -> invert ->
    quantize -> build_plan -> apply): the b200 result is the Python
    backend's, bit for bit, for every digit count the acceptance suite uses."""
    grid, _, ainv, rhs = cells(11)
    for m in (1, 2, 3, 5, 6):
        plan = invop.build_plan(invop.quantize(ainv, m))
        y, counts = invop.apply(plan, rhs)
        out_r = np.zeros(plan.n)
        counts_r = _fallback.plan_apply(plan.col_ptr, plan.group_coeff, plan.group_ptr,
                                        plan.entry_rows, plan.entry_signs,
                                        np.ascontiguousarray(rhs, dtype=np.float64), out_r)
        assert y.tobytes() == out_r.tobytes(), m
        assert counts.as_tuple() == tuple(counts_r), m
