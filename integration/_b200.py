"""INVOP_BACKEND=b200 — the reference's kernel seam bound to libinvop_b200.so.

Drop this file into the reference package as `invop/_kernels/_b200.py` and
add one branch to `invop/_kernels/__init__.py:14-34` (see
`integration/enable_b200.py`, which applies exactly that edit to a copy):

    elif _requested == "b200":
        from . import _b200 as _impl
        BACKEND = "b200"

The four module-level names the seam binds (`_kernels/__init__.py:36-39`)
keep the reference's signatures and contracts (`_native.pyx:15-149`):

  plan_apply(col_ptr, group_coeff, group_ptr, entry_rows, entry_signs, x, out)
      accumulates into the caller's `out` and returns (multiplications,
      additions). The CSC group tables are turned into a device plan once per
      ApplyPlan (tables are immutable, applyplan.py:36-39) and every call runs
      the ordered fp64 kernel (k2_ordered): each row receives its terms in
      ascending column order exactly like the reference, so `out` is bitwise
      equal to the compiled and Python backends.
  naive_apply(col_ptr, rows, vals, x, out)   — same arithmetic (vals are
      signed mant * 10^-m; negation is exact), same device path.
  dense_matvec(mat, x, out)                  — device fp64 GEMV, ascending j,
      no FMA (bitwise equal).
  relax_solve(...)                           — the SOR/Gauss-Seidel baseline
      is not part of the inverse-operator apply this library replaces; it
      stays on the reference's own compiled kernel.

Only ctypes and numpy are needed on the reference side; the library path
comes from INVOP_B200_LIB (default: the in-tree build next to this repo).
The library needs a CUDA device: every call raises if none is visible.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import weakref
from pathlib import Path

import numpy as np

def _default_lib() -> str:
    # the in-tree build of the repository this copy was staged from
    for d in Path(__file__).resolve().parents:
        cand = d / "paper_1602_00001_b200" / "libinvop_b200.so"
        if cand.exists():
            return str(cand)
    return "libinvop_b200.so"


_lib = C.CDLL(os.environ.get("INVOP_B200_LIB") or _default_lib())
_vp, _i64, _int = C.c_void_p, C.c_int64, C.c_int
_lib.invop_last_error.restype = C.c_char_p
_lib.invop_plan_from_csc_host.argtypes = [_i64, _int] + [_vp] * 5 + [_i64, _i64, _vp, C.POINTER(_vp)]
_lib.invop_apply_host_acc.argtypes = [_vp, _vp, _vp, _i64, _vp]
_lib.invop_dense_matvec_host.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _vp]
_lib.invop_plan_destroy.argtypes = [_vp]
for _f in ("invop_plan_from_csc_host", "invop_apply_host_acc", "invop_dense_matvec_host",
           "invop_plan_destroy"):
    getattr(_lib, _f).restype = _int


def _check(rc: int, what: str) -> None:
    if rc:
        msg = (_lib.invop_last_error() or b"").decode("utf-8", "replace")
        raise ValueError("libinvop_b200 %s failed (%d): %s" % (what, rc, msg))


def _digits_of(coeff: np.ndarray):
    """(digits, |mantissa|) such that fl(|mantissa| * 10.0**-digits) reproduces
    every coefficient bit for bit (quant.py:42-45, applyplan.py:168). The
    device kernel recomputes the coefficient that way, so its products
    coeff * x_j are the reference's."""
    c = np.abs(np.asarray(coeff, dtype=np.float64))
    for m in range(0, 13):
        scale = 10.0 ** (-m)
        mag = np.rint(c * (10.0 ** m))
        if mag.size and mag.max() > 2.0 ** 53:
            break
        if np.array_equal(mag * scale, c):
            return m, mag.astype(np.int64)
    raise ValueError("coefficients are not decimally quantized values (|v| * 10^-m, m <= 12)")


class _Plan:
    __slots__ = ("h", "n", "G", "E", "_fin", "__weakref__")

    def __init__(self, h, n, G, E):
        self.h, self.n, self.G, self.E = h, n, G, E
        self._fin = weakref.finalize(self, _lib.invop_plan_destroy, h)


_plans: dict = {}


def _device_plan(col_ptr, coeff, group_ptr, entry_rows, entry_signs) -> _Plan:
    # an ApplyPlan's tables are read-only (applyplan.py:36-39): key those by
    # their buffers (the entry keeps the arrays alive so addresses stay
    # unique); tables a caller may still mutate are keyed by their contents
    tabs = (col_ptr, coeff, group_ptr, entry_rows, entry_signs)
    if any(a.flags.writeable for a in tabs):
        dig = hashlib.blake2b(digest_size=16)
        for a in tabs:
            dig.update(np.int64(a.size).tobytes())
            dig.update(a.tobytes())
        key = ("content", dig.digest())
    else:
        key = tuple((a.__array_interface__["data"][0], a.size) for a in tabs)
    hit = _plans.get(key)
    if hit is not None:
        return hit[0]
    n = col_ptr.size - 1
    m, mag = _digits_of(coeff)
    h = _vp()
    _check(_lib.invop_plan_from_csc_host(
        n, m, col_ptr.ctypes.data, mag.ctypes.data, group_ptr.ctypes.data, entry_rows.ctypes.data,
        entry_signs.ctypes.data, coeff.size, entry_rows.size, None, C.byref(h)), "plan_from_csc")
    plan = _Plan(h, n, coeff.size, entry_rows.size)
    if len(_plans) > 64:
        _plans.clear()
    _plans[key] = (plan, (col_ptr, coeff, group_ptr, entry_rows, entry_signs))
    return plan


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def plan_apply(col_ptr, group_coeff, group_ptr, entry_rows, entry_signs, x, out):
    """_native.pyx:15-49 on the device (ordered fp64, bitwise equal)."""
    col_ptr = _c(col_ptr, np.int64)
    group_coeff = _c(group_coeff, np.float64)
    group_ptr = _c(group_ptr, np.int64)
    entry_rows = _c(entry_rows, np.int32)
    entry_signs = _c(entry_signs, np.int8)
    xv = _c(x, np.float64)
    n = col_ptr.size - 1
    if xv.shape != (n,) or out.shape != (n,) or out.dtype != np.float64:
        raise ValueError("x and out must be float64 vectors of length %d" % n)
    mults = int(col_ptr[n] - col_ptr[0]) if n >= 0 else 0
    adds = int(group_ptr[col_ptr[n]] - group_ptr[col_ptr[0]]) if group_ptr.size else 0
    if n == 0 or group_coeff.size == 0:
        return mults, adds
    plan = _device_plan(col_ptr, group_coeff, group_ptr, entry_rows, entry_signs)
    y = _c(out, np.float64).copy()
    _check(_lib.invop_apply_host_acc(plan.h, xv.ctypes.data, y.ctypes.data, 1, None), "apply")
    out[:] = y
    return mults, adds


def naive_apply(col_ptr, rows, vals, x, out):
    """_native.pyx:52-72: one product and one addition per stored nonzero, as
    a plan with one group per entry (same device kernel, same bits)."""
    col_ptr = _c(col_ptr, np.int64)
    rows = _c(rows, np.int32)
    vals = _c(vals, np.float64)
    n = col_ptr.size - 1
    ops = int(col_ptr[n] - col_ptr[0]) if n >= 0 else 0
    if n == 0 or vals.size == 0:
        return ops, ops
    # group g = entry g: group_ptr = 0..E, col_ptr indexes entries directly
    gptr = np.arange(vals.size + 1, dtype=np.int64)
    signs = np.where(vals > 0, 1, -1).astype(np.int8)
    plan_apply(col_ptr, np.abs(vals), gptr, rows, signs, x, out)
    return ops, ops


def dense_matvec(mat, x, out):
    """_native.pyx:75-92 on the device: acc = m[r,0]*x[0], then += in
    ascending j, no FMA; returns (rows*cols, rows*(cols-1))."""
    m = _c(mat, np.float64)
    xv = _c(x, np.float64)
    rows, cols = m.shape
    y = np.empty(rows, dtype=np.float64)
    _check(_lib.invop_dense_matvec_host(m.ctypes.data, rows, cols, cols, xv.ctypes.data,
                                        y.ctypes.data, None), "dense_matvec")
    out[:] = y
    return rows * cols, rows * (cols - 1)


def relax_solve(*args, **kwargs):
    """Out of scope (the SOR baseline, iterative.py): the reference's own kernel."""
    try:
        from . import _native as impl
    except ImportError:
        from . import _fallback as impl
    return impl.relax_solve(*args, **kwargs)
