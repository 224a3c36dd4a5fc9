"""Plan construction and the counted fast apply (A4-A8) on the device.

API parity with /root/reference/pkg/src/invop/applyplan.py: `ApplyPlan`
(:42-98), `build_plan` (:116-172), `apply` (:175-191),
`apply_naive_quantized` (:194-209), `CostPrediction` /
`predict_direct_costs` (:101-113, :212-225).

An ApplyPlan owns the quantized operator in the compressed device layout
(`DevicePlan`). The reference's CSC group tables (`col_ptr`, `group_ptr`,
`entry_rows`, ...) are still available as attributes: they are built on the
device from the codes the first time one of them is read. Constructing an
ApplyPlan from tables (the reference's dataclass constructor) validates them
exactly like the reference and scatters them into codes on the device.

`apply(plan, x)` defaults to the reference contract: fp64, every output row
accumulated in ascending column order, bitwise equal to the reference's
`apply` and `apply_naive_quantized`. `precision="f32"` selects the fp32 I/O kernels,
which compute every row as an EXACT integer dot product of the mantissas with
x in 23-bit fixed point (one multiplication by 10^-m 2^-e per row). Exact
integer sums make the reference's grouping by distinct |mantissa| (one
multiplication per group, the paper's operation-count argument) unnecessary
for accuracy, and on the GPU a multiply costs no more than the add it would
save, so the device never groups: the `OpCounters` returned are the
reference's PLANNED counts (G distinct values per column, E entries), computed
on the device from the codes, not operations the kernels executed. Device
tensors in give device tensors out, without a host synchronisation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as dev
from . import _lib as L
from ._plan import DevicePlan
from .counting import OpCounters
from .quant import QuantizedMatrix

__all__ = [
    "ApplyPlan",
    "OpCounters",
    "CostPrediction",
    "build_plan",
    "apply",
    "apply_many",
    "apply_naive_quantized",
    "predict_direct_costs",
]

_TABLES = ("col_ptr", "group_abs_mantissa", "group_coeff", "group_ptr", "entry_rows", "entry_signs")


def _frozen(arr, dtype) -> np.ndarray:
    out = np.ascontiguousarray(arr, dtype=dtype)
    out.setflags(write=False)
    return out


def _validate_tables(n, col_ptr, gabs, gcoeff, gptr, rows, signs):
    """The reference's table validation (applyplan.py:60-90)."""
    groups = gabs.shape[0]
    if col_ptr.shape != (n + 1,) or col_ptr[0] != 0 or col_ptr[-1] != groups:
        raise ValueError("column pointer table inconsistent with group count")
    if np.any(np.diff(col_ptr) < 0) or np.any(np.diff(gptr) < 0):
        raise ValueError("pointer tables must be non-decreasing")
    if gptr.shape != (groups + 1,) or gptr[0] != 0 or gptr[-1] != rows.shape[0]:
        raise ValueError("group pointer table inconsistent with entry count")
    if gcoeff.shape != (groups,):
        raise ValueError("coefficient table size mismatch")
    if groups and gabs.min() <= 0:
        raise ValueError("group mantissas must be positive magnitudes")
    if rows.shape != signs.shape:
        raise ValueError("entry tables size mismatch")
    if signs.size and not np.isin(signs, (-1, 1)).all():
        raise ValueError("entry signs must be +1 or -1")


class ApplyPlan:
    """Quantized operator ready for counted fast apply on the device."""

    def __init__(self, n, scale_digits, col_ptr=None, group_abs_mantissa=None, group_coeff=None,
                 group_ptr=None, entry_rows=None, entry_signs=None, *, _dplan=None):
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "scale_digits", int(scale_digits))
        object.__setattr__(self, "_tables", None)
        object.__setattr__(self, "_dplan", _dplan)
        if _dplan is not None:
            return
        tabs = (
            _frozen(col_ptr, np.int64),
            _frozen(group_abs_mantissa, np.int64),
            _frozen(group_coeff, np.float64),
            _frozen(group_ptr, np.int64),
            _frozen(entry_rows, np.int32),
            _frozen(entry_signs, np.int8),
        )
        _validate_tables(self.n, *tabs)
        object.__setattr__(self, "_tables", dict(zip(_TABLES, tabs)))
        object.__setattr__(
            self, "_dplan",
            DevicePlan.from_csc(self.n, self.scale_digits, tabs[0], tabs[1], tabs[3], tabs[4], tabs[5]),
        )

    def __setattr__(self, name, value):
        raise AttributeError("ApplyPlan is immutable")

    def __repr__(self):
        d = self._dplan
        return "ApplyPlan(n=%d, scale_digits=%d, code_bytes=%d)" % (
            self.n, self.scale_digits, d.code_bytes)

    # reference table attributes, materialised lazily from the device codes
    def _table(self, name):
        if self._tables is None:
            raw = self._dplan.csc_tables()
            tabs = {k: _frozen(raw[k], v.dtype) for k, v in zip(_TABLES, (
                np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.float64),
                np.zeros(0, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int8)))}
            object.__setattr__(self, "_tables", tabs)
        return self._tables[name]

    col_ptr = property(lambda self: self._table("col_ptr"))
    group_abs_mantissa = property(lambda self: self._table("group_abs_mantissa"))
    group_coeff = property(lambda self: self._table("group_coeff"))
    group_ptr = property(lambda self: self._table("group_ptr"))
    entry_rows = property(lambda self: self._table("entry_rows"))
    entry_signs = property(lambda self: self._table("entry_signs"))

    @property
    def device_plan(self) -> DevicePlan:
        return self._dplan

    @property
    def planned_multiplications(self) -> int:
        return self._dplan.counts()[0]

    @property
    def planned_additions(self) -> int:
        return self._dplan.counts()[1]

    def counters(self) -> OpCounters:
        m, a = self._dplan.counts()
        return OpCounters(int(m), int(a))


@dataclass(frozen=True)
class CostPrediction:
    """Reference cost-model values reported next to measured counts."""

    direct_products: float
    direct_sums: float
    iterative_total: float
    iterations: float

    def __post_init__(self):
        for name in ("direct_products", "direct_sums", "iterative_total", "iterations"):
            if getattr(self, name) < 0:
                raise ValueError("%s must be non-negative" % name)


def build_plan(q: QuantizedMatrix) -> ApplyPlan:
    """Encode a quantized matrix for the device apply (deterministic)."""
    if q.n == 0:
        return _empty_plan(q.scale_digits)
    return ApplyPlan(n=q.n, scale_digits=q.scale_digits, _dplan=q.device_plan())


def _empty_plan(digits):
    return _EmptyPlan(digits)


class _EmptyPlan:
    """n = 0 operator: nothing lives on the device."""

    def __init__(self, digits):
        self.n = 0
        self.scale_digits = digits
        self.col_ptr = _frozen(np.zeros(1), np.int64)
        self.group_abs_mantissa = _frozen(np.zeros(0), np.int64)
        self.group_coeff = _frozen(np.zeros(0), np.float64)
        self.group_ptr = _frozen(np.zeros(1), np.int64)
        self.entry_rows = _frozen(np.zeros(0), np.int32)
        self.entry_signs = _frozen(np.zeros(0), np.int8)
        self.planned_multiplications = 0
        self.planned_additions = 0

    def counters(self):
        return OpCounters(0, 0)


_PRECISION = {"f64": L.MODE_ORDERED, "ordered": L.MODE_ORDERED, "f32": L.MODE_FAST,
              "fast": L.MODE_FAST}


def _mode(precision: str) -> int:
    try:
        return _PRECISION[precision]
    except KeyError:
        raise ValueError("precision must be one of %s" % sorted(_PRECISION)) from None


def apply(plan, x, *, precision: str = "f64") -> tuple:
    """Execute the plan on x. Returns (y, OpCounters).

    precision="f64" (default): bitwise equal to the reference apply.
    precision="f32": fp32 I/O, exact integer row sums (max relative error ~1e-6).
    The counters are the reference's planned counts (applyplan.py:92-98).
    x may be a host vector (numpy / list; result is a float64 numpy array,
    like the reference) or a CUDA tensor (result stays on the device).
    """
    mode = _mode(precision)
    if isinstance(plan, _EmptyPlan):
        vec = np.ascontiguousarray(x, dtype=np.float64)
        if vec.shape != (0,):
            raise ValueError("vector length %s does not match n=0" % (vec.shape,))
        return np.zeros(0), OpCounters(0, 0)
    t = dev.torch()
    if isinstance(x, t.Tensor) and x.is_cuda:
        if tuple(x.shape) != (plan.n,):
            raise ValueError("vector length %s does not match n=%d" % (tuple(x.shape), plan.n))
        return plan.device_plan.apply_device(x, mode=mode), plan.counters()
    vec = np.ascontiguousarray(x, dtype=np.float64)
    if vec.shape != (plan.n,):
        raise ValueError("vector length %s does not match n=%d" % (vec.shape, plan.n))
    return plan.device_plan.apply_host(vec, mode=mode), plan.counters()


def apply_many(plan, X, *, precision: str = "f32"):
    """Multi-RHS apply: X is [k, n] (k right-hand sides, RHS-major); returns
    Y [k, rows] (same kind of container as X) and the per-RHS counters."""
    mode = _mode(precision)
    t = dev.torch()
    if isinstance(X, t.Tensor) and X.is_cuda:
        if X.dim() != 2 or X.shape[1] != plan.n:
            raise ValueError("X must be [k, %d]" % plan.n)
        return plan.device_plan.apply_device(X, mode=mode), plan.counters()
    Xh = np.ascontiguousarray(X, dtype=np.float64)
    if Xh.ndim != 2 or Xh.shape[1] != plan.n:
        raise ValueError("X must be [k, %d]" % plan.n)
    return plan.device_plan.apply_host(Xh, mode=mode), plan.counters()


def apply_naive_quantized(q: QuantizedMatrix, x) -> tuple:
    """Oracle-order apply of the reference (ascending columns, one product and
    one addition per nonzero), on the device; counters (E, E)."""
    vec = np.ascontiguousarray(x, dtype=np.float64)
    if vec.shape != (q.n,):
        raise ValueError("vector length %s does not match n=%d" % (vec.shape, q.n))
    if q.n == 0:
        return np.zeros(0), OpCounters(0, 0)
    dplan = q.device_plan()
    y = dplan.apply_host(vec, mode=L.MODE_ORDERED)
    nz = dplan.counts()[1]
    return y, OpCounters(int(nz), int(nz))


def predict_direct_costs(m: int, n_total: int) -> CostPrediction:
    """Eq. 9/10 of the paper with the iterative predictions beside them
    (reference applyplan.py:212-225)."""
    from .iterative import predict_iterations, predict_iterative_total

    if m < 1:
        raise ValueError("m must be at least 1, got %d" % m)
    if n_total < 1:
        raise ValueError("n_total must be at least 1, got %d" % n_total)
    factor = float(m) ** 2.5 * n_total
    return CostPrediction(
        direct_products=2.5 * factor,
        direct_sums=14.2 * factor,
        iterative_total=predict_iterative_total(n_total, m),
        iterations=predict_iterations(n_total, m),
    )
