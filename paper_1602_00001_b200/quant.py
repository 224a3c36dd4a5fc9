"""Decimal quantization of operators to integer mantissas (A1-A3, A9).

API parity with /root/reference/pkg/src/invop/quant.py: `quantize`
(:48-65), `QuantizedMatrix` (:22-45), `dequantize` (:68-70),
`sparsity_stats` (:73-82), `MANTISSA_LIMIT` (:19).

A QuantizedMatrix produced by `quantize` lives on the device in the
compressed byte-plane layout (csrc/common.cuh); its `mantissas` attribute is
materialised on the host only when read. Constructing one from a host int64
array (the reference constructor) keeps the array and encodes it on device
the first time a plan is built.
"""

from __future__ import annotations

import numpy as np

from ._plan import DevicePlan
from .dense import DenseMatrix

MANTISSA_LIMIT = 2 ** 53

_MISSING = object()


class QuantizedMatrix:
    """Integer-mantissa matrix at decimal scale 10^(-scale_digits).

    Immutable; `mantissas` is a read-only int64 [n x n] array.
    """

    __slots__ = ("n", "scale_digits", "_mant", "_dplan", "__weakref__")

    def __init__(self, n: int, scale_digits: int, mantissas=_MISSING, *, _dplan=None):
        if scale_digits < 0:
            raise ValueError("scale_digits must be non-negative")
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "scale_digits", int(scale_digits))
        object.__setattr__(self, "_dplan", _dplan)
        if mantissas is _MISSING:
            if _dplan is None:
                raise TypeError("QuantizedMatrix needs mantissas")
            object.__setattr__(self, "_mant", None)
            return
        raw = np.asarray(mantissas)
        if not np.issubdtype(raw.dtype, np.integer):
            raise ValueError("mantissas must be integers, got dtype %s" % raw.dtype)
        mant = np.ascontiguousarray(raw, dtype=np.int64)
        if mant.shape != (self.n, self.n):
            raise ValueError("mantissas shape %s does not match n=%d" % (mant.shape, self.n))
        mant.setflags(write=False)
        object.__setattr__(self, "_mant", mant)

    def __setattr__(self, name, value):
        raise AttributeError("QuantizedMatrix is immutable")

    def __repr__(self):
        return "QuantizedMatrix(n=%d, scale_digits=%d)" % (self.n, self.scale_digits)

    @property
    def scale(self) -> float:
        """The exact double every consumer multiplies mantissas by."""
        return 10.0 ** (-self.scale_digits)

    @property
    def mantissas(self) -> np.ndarray:
        if self._mant is None:
            m = self._dplan.decode().cpu().numpy()
            m.setflags(write=False)
            object.__setattr__(self, "_mant", m)
        return self._mant

    def device_plan(self) -> DevicePlan:
        """The compressed device encoding (built on first use)."""
        if self._dplan is None:
            object.__setattr__(
                self, "_dplan", DevicePlan.from_mantissas(self._mant, self.scale_digits)
            )
        return self._dplan


def quantize(mat: DenseMatrix, digits: int) -> QuantizedMatrix:
    """Round every entry to `digits` decimal places, half away from zero, on
    the device (reference quant.py:48-65; same MantissaOverflowError contract)."""
    if not 0 <= digits <= 12:
        raise ValueError("digits must be in 0..12, got %d" % digits)
    if mat.n == 0:
        return QuantizedMatrix(n=0, scale_digits=digits, mantissas=np.zeros((0, 0), np.int64))
    dplan = DevicePlan.from_entries(mat.entries, digits)
    return QuantizedMatrix(n=mat.n, scale_digits=digits, _dplan=dplan)


def dequantize(q: QuantizedMatrix) -> DenseMatrix:
    """The exact doubles the apply uses: mantissa * 10^-m (reference :68-70)."""
    return DenseMatrix(n=q.n, entries=q.mantissas.astype(np.float64) * q.scale)


def sparsity_stats(q: QuantizedMatrix) -> tuple:
    """(nonzero count, per-column count of distinct nonzero |mantissa|),
    computed on device from the codes (reference :73-82)."""
    if q.n == 0:
        return 0, []
    distinct, nonzero = q.device_plan().column_stats()
    return int(nonzero.sum()), [int(v) for v in distinct]
