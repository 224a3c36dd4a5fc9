"""ctypes binding of libinvop_b200.so (the C ABI declared in include/invop_b200.h).

There is no fallback: if the shared library is missing or fails to load, the
import raises. Status codes are mapped onto the reference's exception
hierarchy (/root/reference/pkg/src/invop/errors.py:4-25).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import (
    CapacityError,
    InvopError,
    MantissaOverflowError,
    SingularMatrixError,
)

# INVOP_LIB_PATH: another build of the same library (A/B timing of kernel
# revisions on one box); the default is the in-tree build
LIB_PATH = Path(os.environ.get("INVOP_LIB_PATH") or
                Path(__file__).resolve().parent / "libinvop_b200.so").resolve()

OK = 0
E_VALUE = 1
E_OVERFLOW = 2
E_CAPACITY = 3
E_SINGULAR = 4
E_CUDA = 5
E_UNSUPPORTED = 6

F32 = 0
F64 = 1
MODE_FAST = 0
MODE_ORDERED = 1

_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_pi64 = C.POINTER(C.c_int64)
_pint = C.POINTER(C.c_int)

# name -> argtypes (restype is int except invop_last_error / invop_apply_kernel: char*)
SIGNATURES = {
    "invop_abi_version": [],
    "invop_quantize": [_vp, _i64, _i64, _i64, _int, _vp, _i64, _pi64, _vp],
    "invop_plan_create": [_vp, _i64, _i64, _i64, _i64, _int, _vp, C.POINTER(_vp)],
    "invop_plan_from_f64": [_vp, _i64, _i64, _i64, _i64, _int, _pi64, _vp, C.POINTER(_vp)],
    "invop_plan_from_csc": [_i64, _int, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, C.POINTER(_vp)],
    "invop_plan_from_csc_host": [_i64, _int, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, C.POINTER(_vp)],
    "invop_apply_host_acc": [_vp, _vp, _vp, _i64, _vp],
    "invop_dense_matvec_host": [_vp, _i64, _i64, _i64, _vp, _vp, _vp],
    "invop_plan_destroy": [_vp],
    "invop_plan_info": [_vp, _pi64, _pi64, _pi64, _pint, _pint, _pint, _pi64, _pi64],
    "invop_plan_counts": [_vp, _pi64, _pi64, _vp],
    "invop_plan_column_stats": [_vp, _vp, _vp, _vp],
    "invop_plan_decode": [_vp, _vp, _i64, _vp],
    "invop_plan_decode_rows": [_vp, _vp, _i64, _vp, _i64, _vp],
    "invop_plan_get_planes": [_vp, _vp, _vp],
    "invop_plan_from_planes": [_vp, _int, _int, _i64, _i64, _i64, _int, _vp, C.POINTER(_vp)],
    "invop_plan_csc": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _pi64, _pi64, _vp],
    "invop_apply_grouped_csc": [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "invop_apply": [_vp, _vp, _i64, _vp, _i64, _i64, _int, _int, _vp],
    "invop_apply_host": [_vp, _vp, _vp, _i64, _int, _vp],
    "invop_apply_sharded": [_vp, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _int, _int, _vp],
    "invop_unshard": [_vp, _int, _vp, _i64, _i64, _vp, _i64, _int, _vp],
    "invop_apply_naive": [_vp, _vp, _vp, _i64, _vp],
    "invop_plan_apply_bytes": [_vp, _i64, _int, _pi64, _vp],
    "invop_plan_tensor_ops": [_vp, _i64, _int, _pi64, _vp],
    "invop_apply_kernel": [_vp, _i64, _int],
    "invop_operator_create": [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_vp)],
    "invop_operator_factor": [_vp, _vp],
    "invop_operator_destroy": [_vp],
    "invop_construct_rows": [_vp, _i64, _i64, _int, _vp, C.POINTER(_vp)],
    "invop_construct_rows_f64": [_vp, _i64, _i64, _vp, _i64, _vp],
    "invop_dense_invert": [_vp, _i64, _vp, C.c_double, _vp],
    "invop_dense_matvec": [_vp, _i64, _i64, _i64, _vp, _vp, _vp],
}


def _load():
    lib = C.CDLL(str(LIB_PATH))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.invop_last_error.argtypes = []
    lib.invop_last_error.restype = C.c_char_p
    lib.invop_apply_kernel.restype = C.c_char_p
    lib.invop_launch_count.argtypes = []
    lib.invop_launch_count.restype = C.c_int64
    return lib


class _Library:
    """libinvop_b200.so, dlopen'ed on first use (importing the package only
    checks that it is built: modules that need no device code, e.g. the
    workload definitions in configs/grid, stay free of the native library)."""

    _cdll = None

    def _get(self):
        if _Library._cdll is None:
            _Library._cdll = _load()
        return _Library._cdll

    def __getattr__(self, name):
        return getattr(self._get(), name)


if not LIB_PATH.exists():
    raise ImportError(
        "libinvop_b200.so is not built (%s); run `python paper_1602_00001_b200/build.py` "
        "or __graft_entry__.build()" % LIB_PATH
    )
lib = _Library()


def loaded() -> bool:
    """True once the native library has been dlopen'ed in this process."""
    return _Library._cdll is not None


def last_error() -> str:
    msg = lib.invop_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Raise the reference-hierarchy exception for a non-zero status."""
    if rc == OK:
        return
    msg = last_error()
    if what:
        msg = "%s: %s" % (what, msg)
    if rc == E_VALUE:
        raise ValueError(msg)
    if rc == E_OVERFLOW:
        raise MantissaOverflowError(msg)
    if rc == E_CAPACITY:
        raise CapacityError(msg)
    if rc == E_SINGULAR:
        raise SingularMatrixError(msg)
    if rc == E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise InvopError("CUDA failure (%d): %s" % (rc, msg))


def exported_symbols() -> list:
    return sorted(list(SIGNATURES) + ["invop_last_error", "invop_launch_count"])


def header_symbols() -> list:
    """Function names declared in include/invop_b200.h."""
    import re

    hdr = Path(__file__).resolve().parent.parent / "include" / "invop_b200.h"
    text = hdr.read_text()
    return sorted(set(re.findall(r"\b(invop_[a-z0-9_]+)\s*\(", text)))


def ptr(x) -> int:
    """Raw address of a torch tensor / numpy array / int (0 for None)."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError("cannot take the address of %r" % type(x).__name__)


os.environ.setdefault("INVOP_B200_LIB", str(LIB_PATH))
