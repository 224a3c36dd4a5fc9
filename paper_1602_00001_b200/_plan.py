"""DevicePlan: owner of one `invop_plan*` (compressed device layout of a
quantized operator shard) and the Python side of every plan-level C-ABI call.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _device as dev
from . import _lib as L


class DevicePlan:
    """Rows [row0, row0+rows) of an n x n quantized operator on the current device."""

    def __init__(self, handle: int, keepalive=None):
        if not handle:
            raise ValueError("null plan handle")
        self._h = C.c_void_p(handle)
        self._finalizer = weakref.finalize(self, L.lib.invop_plan_destroy, C.c_void_p(handle))
        self._keepalive = keepalive
        n, rows, row0, mx = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        digits, cb, sg = C.c_int(), C.c_int(), C.c_int()
        nbytes = C.c_int64()
        L.check(L.lib.invop_plan_info(self._h, C.byref(n), C.byref(rows), C.byref(row0),
                                      C.byref(digits), C.byref(cb), C.byref(sg),
                                      C.byref(nbytes), C.byref(mx)), "plan_info")
        self.n = n.value
        self.rows = rows.value
        self.row0 = row0.value
        self.scale_digits = digits.value
        self.code_bytes = cb.value
        self.is_signed = bool(sg.value)
        self.device_bytes = nbytes.value
        self.max_abs = mx.value
        self._counts = None

    # ----------------------------------------------------------- constructors
    @classmethod
    def from_mantissas(cls, mant, scale_digits: int, row0: int = 0, n: int = None):
        """Encode int64 mantissas (host array or device tensor, rows x n)."""
        t = dev.require_cuda()
        d = dev.to_device(mant, t.int64)
        if d.dim() != 2:
            raise ValueError("mantissas must be 2-D")
        rows, cols = d.shape
        n = cols if n is None else n
        out = C.c_void_p()
        L.check(L.lib.invop_plan_create(L.ptr(d), rows, n, cols, row0, scale_digits,
                                        C.c_void_p(dev.stream_ptr()), C.byref(out)), "plan_create")
        return cls(out.value)

    @classmethod
    def from_entries(cls, entries, digits: int, row0: int = 0, n: int = None):
        """Fused quantize + encode of fp64 entries (host array or device tensor)."""
        t = dev.require_cuda()
        d = dev.to_device(entries, t.float64)
        rows, cols = d.shape
        n = cols if n is None else n
        out = C.c_void_p()
        bad = C.c_int64(-1)
        rc = L.lib.invop_plan_from_f64(L.ptr(d), rows, n, cols, row0, digits, C.byref(bad),
                                       C.c_void_p(dev.stream_ptr()), C.byref(out))
        if rc == L.E_OVERFLOW:
            i, j = divmod(int(bad.value), cols)
            val = float(d[i, j].item())
            from .errors import MantissaOverflowError

            raise MantissaOverflowError(
                "entry (%d, %d) = %r needs mantissa %g at %d digits, beyond 2^53"
                % (i, j, val, abs(val) * 10.0 ** digits, digits)
            )
        L.check(rc, "plan_from_f64")
        return cls(out.value)

    @classmethod
    def from_csc(cls, n, scale_digits, col_ptr, group_abs, group_ptr, entry_rows, entry_signs):
        t = dev.require_cuda()
        cp = dev.to_device(col_ptr, t.int64)
        ga = dev.to_device(group_abs, t.int64)
        gp = dev.to_device(group_ptr, t.int64)
        er = dev.to_device(entry_rows, t.int32)
        es = dev.to_device(entry_signs, t.int8)
        out = C.c_void_p()
        L.check(L.lib.invop_plan_from_csc(n, scale_digits, L.ptr(cp), L.ptr(ga), L.ptr(gp),
                                          L.ptr(er), L.ptr(es), ga.numel(), er.numel(),
                                          C.c_void_p(dev.stream_ptr()), C.byref(out)),
                "plan_from_csc")
        return cls(out.value)

    # ----------------------------------------------------------- queries
    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def counts(self) -> tuple:
        if self._counts is None:
            m, a = C.c_int64(), C.c_int64()
            L.check(L.lib.invop_plan_counts(self._h, C.byref(m), C.byref(a),
                                            C.c_void_p(dev.stream_ptr())), "plan_counts")
            self._counts = (m.value, a.value)
        return self._counts

    def column_stats(self) -> tuple:
        t = dev.require_cuda()
        d = t.empty(2 * max(self.n, 1), dtype=t.int64, device="cuda")
        L.check(L.lib.invop_plan_column_stats(self._h, L.ptr(d), L.ptr(d) + 8 * max(self.n, 1),
                                              C.c_void_p(dev.stream_ptr())), "column_stats")
        h = d.cpu().numpy()
        return h[: self.n].copy(), h[max(self.n, 1): max(self.n, 1) + self.n].copy()

    def apply_kernel(self, nrhs: int = 1, mode: int = 0) -> str:
        """Name of the kernel an apply of `nrhs` right-hand sides launches."""
        return L.lib.invop_apply_kernel(self._h, nrhs, mode).decode()

    def decode(self):
        """int64 mantissas as a device tensor [rows x n]."""
        t = dev.require_cuda()
        out = t.empty((self.rows, self.n), dtype=t.int64, device="cuda")
        if self.rows and self.n:
            L.check(L.lib.invop_plan_decode(self._h, L.ptr(out), self.n,
                                            C.c_void_p(dev.stream_ptr())), "plan_decode")
        return out

    def decode_rows(self, rows):
        """int64 mantissas of the given plan-local rows as a device tensor [len(rows) x n]."""
        t = dev.require_cuda()
        sel = dev.to_device(np.asarray(rows, dtype=np.int64).reshape(-1), t.int64)
        if sel.numel() and (int(sel.min()) < 0 or int(sel.max()) >= self.rows):
            raise ValueError("row index out of range")
        out = t.empty((sel.numel(), self.n), dtype=t.int64, device="cuda")
        if sel.numel() and self.n:
            L.check(L.lib.invop_plan_decode_rows(self._h, L.ptr(sel), sel.numel(), L.ptr(out), self.n,
                                                 C.c_void_p(dev.stream_ptr())), "plan_decode_rows")
        return out

    def csc_tables(self) -> dict:
        t = dev.require_cuda()
        s = C.c_void_p(dev.stream_ptr())
        G, E = C.c_int64(), C.c_int64()
        L.check(L.lib.invop_plan_csc(self._h, None, None, None, None, None, None,
                                     C.byref(G), C.byref(E), s), "plan_csc(size)")
        n = self.n
        col_ptr = t.zeros(n + 1, dtype=t.int64, device="cuda")
        gabs = t.empty(max(G.value, 1), dtype=t.int64, device="cuda")
        gcoeff = t.empty(max(G.value, 1), dtype=t.float64, device="cuda")
        gptr = t.zeros(G.value + 1, dtype=t.int64, device="cuda")
        rows = t.empty(max(E.value, 1), dtype=t.int32, device="cuda")
        signs = t.empty(max(E.value, 1), dtype=t.int8, device="cuda")
        L.check(L.lib.invop_plan_csc(self._h, L.ptr(col_ptr), L.ptr(gabs), L.ptr(gcoeff),
                                     L.ptr(gptr), L.ptr(rows), L.ptr(signs), C.byref(G),
                                     C.byref(E), s), "plan_csc")
        g, e = G.value, E.value
        return {
            "col_ptr": col_ptr.cpu().numpy(),
            "group_abs_mantissa": gabs[:g].cpu().numpy(),
            "group_coeff": gcoeff[:g].cpu().numpy(),
            "group_ptr": gptr.cpu().numpy(),
            "entry_rows": rows[:e].cpu().numpy(),
            "entry_signs": signs[:e].cpu().numpy(),
        }

    # ----------------------------------------------------------- apply
    def apply_device(self, x, y=None, ldy: int = None, *, mode: int = L.MODE_ORDERED):
        """x: device tensor [n] or [k, n]; returns device tensor [rows] / [k, rows]
        (or writes into `y`, RHS t at y[t*ldy :], when given)."""
        t = dev.require_cuda()
        dtype = t.float64 if mode == L.MODE_ORDERED else t.float32
        x = x.to(dtype=dtype).contiguous()
        one = x.dim() == 1
        X = x.view(1, -1) if one else x
        if X.shape[1] != self.n:
            raise ValueError("vector length %d does not match n=%d" % (X.shape[1], self.n))
        k = X.shape[0]
        if y is None:
            y = t.empty((k, self.rows), dtype=dtype, device="cuda")
        elif y.dtype != dtype or not y.is_cuda:
            raise ValueError("y must be a device tensor of %s" % dtype)
        ldy = self.rows if ldy is None else int(ldy)
        if ldy < self.rows or y.numel() < (k - 1) * ldy + self.rows:
            raise ValueError("y is too small for %d right-hand sides" % k)
        L.check(L.lib.invop_apply(self._h, L.ptr(X), self.n, L.ptr(y), ldy, k,
                                  L.F64 if mode == L.MODE_ORDERED else L.F32, mode,
                                  C.c_void_p(dev.stream_ptr())), "apply")
        return y.view(-1) if one else y

    def apply_host(self, x: np.ndarray, mode: int = L.MODE_ORDERED) -> np.ndarray:
        """Host fp64 in, host fp64 out; copies happen inside the C-ABI call."""
        dev.require_cuda()
        X = np.ascontiguousarray(x, dtype=np.float64)
        one = X.ndim == 1
        X2 = X.reshape(1, -1) if one else X
        k = X2.shape[0]
        Y = np.empty((k, self.rows), dtype=np.float64)
        L.check(L.lib.invop_apply_host(self._h, X2.ctypes.data, Y.ctypes.data, k, mode,
                                       C.c_void_p(dev.stream_ptr())), "apply_host")
        return Y.reshape(-1) if one else Y
