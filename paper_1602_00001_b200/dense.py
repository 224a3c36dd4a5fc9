"""Dense matrices, inversion (setup) and the counted dense apply.

API parity with /root/reference/pkg/src/invop/dense.py: `DenseMatrix`
(:19-33), `invert` (:36-62), `residual_check` (:65-71), `apply_dense`
(:74-82), `PIVOT_RTOL` (:16).

`invert` runs on the device: 5-point grid operators (anything carrying a
`stencil`, or a StencilOperator itself) go through the block-tridiagonal
constructor of csrc/construct.cu; any other dense matrix through device
Gauss-Jordan with partial pivoting (csrc/dense.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from . import _lib as L
from .counting import OpCounters
from .errors import SingularMatrixError

PIVOT_RTOL = 1e-13


@dataclass(frozen=True)
class DenseMatrix:
    """Immutable dense N x N real matrix, row-major."""

    n: int
    entries: np.ndarray

    def __post_init__(self):
        ent = np.ascontiguousarray(self.entries, dtype=np.float64)
        if ent.shape != (self.n, self.n):
            raise ValueError("entries shape %s does not match n=%d" % (ent.shape, self.n))
        if not np.isfinite(ent).all():
            raise ValueError("matrix entries must be finite")
        ent.setflags(write=False)
        object.__setattr__(self, "entries", ent)


class DeviceOperator:
    """A 5-point stencil operator resident on the device, factorised once
    (block LU over grid lines) and reused for any set of rows of its inverse."""

    def __init__(self, stencil):
        dev.require_cuda()
        self.stencil = stencil
        self.n = stencil.n
        h = C.c_void_p()
        arrs = [np.ascontiguousarray(getattr(stencil, k), dtype=np.float64)
                for k in ("diag", "w_west", "w_east", "w_south", "w_north")]
        self._arrs = arrs
        L.check(L.lib.invop_operator_create(stencil.nx, stencil.ny, *[a.ctypes.data for a in arrs],
                                            C.c_void_p(dev.stream_ptr()), C.byref(h)),
                "operator_create")
        self._h = h
        import weakref

        self._fin = weakref.finalize(self, L.lib.invop_operator_destroy, C.c_void_p(h.value))

    def factor(self) -> "DeviceOperator":
        L.check(L.lib.invop_operator_factor(self._h, C.c_void_p(dev.stream_ptr())), "factor")
        return self

    def inverse_rows(self, row0: int = 0, rows: int = None):
        """fp64 rows [row0, row0+rows) of the inverse as a device tensor."""
        t = dev.require_cuda()
        rows = self.n - row0 if rows is None else rows
        out = t.empty((rows, self.n), dtype=t.float64, device="cuda")
        L.check(L.lib.invop_construct_rows_f64(self._h, row0, rows, L.ptr(out), self.n,
                                               C.c_void_p(dev.stream_ptr())), "construct_rows_f64")
        return out

    def quantized_rows(self, digits: int, row0: int = 0, rows: int = None):
        """Rows of the inverse quantized to `digits` straight into a device plan."""
        from ._plan import DevicePlan

        rows = self.n - row0 if rows is None else rows
        h = C.c_void_p()
        L.check(L.lib.invop_construct_rows(self._h, row0, rows, digits,
                                           C.c_void_p(dev.stream_ptr()), C.byref(h)),
                "construct_rows")
        return DevicePlan(h.value)


def _stencil_of(a):
    from .grid import StencilOperator

    if isinstance(a, StencilOperator):
        return a
    return getattr(a, "stencil", None)


def invert(a) -> DenseMatrix:
    """Invert a square matrix container (anything with .n and .entries, or a
    StencilOperator) on the device. Raises SingularMatrixError when a pivot
    falls below PIVOT_RTOL * max|entry| (reference dense.py:36-62)."""
    st = _stencil_of(a)
    n = a.n
    if st is not None:
        ent = None
        scale = max(float(np.abs(getattr(st, k)).max()) if n else 0.0
                    for k in ("diag", "w_west", "w_east", "w_south", "w_north"))
    else:
        ent = np.asarray(a.entries, dtype=np.float64)
        scale = float(np.abs(ent).max()) if n else 0.0
    if scale == 0.0:
        raise SingularMatrixError("matrix is identically zero")
    if st is not None:
        inv = DeviceOperator(st).factor().inverse_rows()
        return DenseMatrix(n=n, entries=inv.cpu().numpy())
    t = dev.require_cuda()
    d = dev.to_device(ent, t.float64)
    out = t.empty((n, n), dtype=t.float64, device="cuda")
    rc = L.lib.invop_dense_invert(L.ptr(d), n, L.ptr(out), PIVOT_RTOL * scale,
                                  C.c_void_p(dev.stream_ptr()))
    if rc == L.E_SINGULAR:
        raise SingularMatrixError(
            "pivot below threshold %.3e; matrix is singular to working precision"
            % (PIVOT_RTOL * scale)
        )
    L.check(rc, "dense_invert")
    return DenseMatrix(n=n, entries=out.cpu().numpy())


def residual_check(a, ainv) -> float:
    """Max-norm of A * Ainv - I (reference dense.py:65-71); a diagnostic."""
    if a.n != ainv.n:
        raise ValueError("dimension mismatch: %d vs %d" % (a.n, ainv.n))
    prod = np.asarray(a.entries) @ np.asarray(ainv.entries)
    np.fill_diagonal(prod, np.diagonal(prod) - 1.0)
    return float(np.abs(prod).max())


def apply_dense(m: DenseMatrix, x) -> tuple:
    """Conventional dense product, ascending-column fp64 accumulation on the
    device (bitwise equal to the reference); counters N*N and N*(N-1)."""
    vec = np.ascontiguousarray(x, dtype=np.float64)
    if vec.shape != (m.n,):
        raise ValueError("vector length %s does not match n=%d" % (vec.shape, m.n))
    t = dev.require_cuda()
    dm = dev.to_device(m.entries, t.float64)
    dx = dev.to_device(vec, t.float64)
    dy = t.empty(m.n, dtype=t.float64, device="cuda")
    L.check(L.lib.invop_dense_matvec(L.ptr(dm), m.n, m.n, m.n, L.ptr(dx), L.ptr(dy),
                                     C.c_void_p(dev.stream_ptr())), "dense_matvec")
    return dy.cpu().numpy(), OpCounters(m.n * m.n, m.n * (m.n - 1) if m.n else 0)
