"""CPU: the C-ABI library loads and exports every declared symbol; host-side
logic of the package (operators, validation, configs) without a GPU."""

import ctypes as C

import numpy as np
import pytest

import paper_1602_00001_b200 as invop
from paper_1602_00001_b200 import _lib


def test_library_exports_header_symbols():
    declared = set(_lib.header_symbols())
    assert declared, "no symbols parsed from include/invop_b200.h"
    lib = C.CDLL(str(_lib.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.exported_symbols())
    assert _lib.lib.invop_abi_version() == 1


def test_error_paths_without_gpu():
    # argument validation happens before any device work
    out = C.c_void_p()
    rc = _lib.lib.invop_plan_create(None, 2, 3, 3, 2, 1, None, C.byref(out))
    assert rc == _lib.E_VALUE and "geometry" in _lib.last_error()
    rc = _lib.lib.invop_plan_create(None, 1, 1, 1, 0, -1, None, C.byref(out))
    assert rc == _lib.E_VALUE
    with pytest.raises(ValueError):
        _lib.check(_lib.E_VALUE)
    with pytest.raises(invop.MantissaOverflowError):
        _lib.check(_lib.E_OVERFLOW)
    with pytest.raises(invop.SingularMatrixError):
        _lib.check(_lib.E_SINGULAR)
    with pytest.raises(invop.CapacityError):
        _lib.check(_lib.E_CAPACITY)
    assert issubclass(invop.MantissaOverflowError, invop.InvopError)


def test_reference_dense_operators(golden):
    g = golden("grid_cases")
    opv = invop.build_variable(invop.Grid2D(6, 5), invop.CoefficientField(g["var_beta"]))
    assert np.array_equal(opv.entries, g["var_entries"])
    with pytest.raises(invop.CapacityError):
        invop.build_uniform(invop.Grid2D(91, 91))
    assert invop.MAX_DENSE_N == 8192


def test_uniform_interior_is_interior_block():
    n = 6
    full = invop.build_uniform(invop.Grid2D(n + 2, n + 2))
    mask = ~full.is_boundary
    block = full.entries[np.ix_(mask, mask)]
    assert np.array_equal(invop.uniform_interior(n).to_dense(), block)


def test_variable_interior_properties():
    st = invop.variable_interior(16, seed=104)
    a = st.to_dense()
    assert np.allclose(np.diag(a), 1.0)
    off = a - np.diag(np.diag(a))
    assert (off <= 0).all()
    # weakly diagonally dominant M-matrix with strict dominance next to the boundary
    rows = -off.sum(axis=1)
    assert (rows <= 1.0 + 1e-12).all() and (rows < 1.0 - 1e-6).any()
    # symmetrizable: a diagonal D with D*A symmetric exists (the control-volume areas)
    assert np.abs(a - a.T).max() > 1e-3
    from paper_1602_00001_b200.grid import nonuniform_spacing

    h = nonuniform_spacing(16)
    assert abs(h.sum() - 1.0) < 1e-15


def test_quantized_matrix_validation():
    with pytest.raises(ValueError):
        invop.QuantizedMatrix(n=2, scale_digits=-1, mantissas=np.zeros((2, 2), dtype=np.int64))
    with pytest.raises(ValueError):
        invop.QuantizedMatrix(n=2, scale_digits=2, mantissas=np.zeros((2, 2)))
    with pytest.raises(ValueError):
        invop.QuantizedMatrix(n=3, scale_digits=2, mantissas=np.zeros((2, 2), dtype=np.int64))
    q = invop.QuantizedMatrix(n=1, scale_digits=2, mantissas=np.array([[12]]))
    assert q.scale == 10.0 ** -2
    assert invop.dequantize(q).entries[0, 0] == 12 * 10.0 ** -2
    with pytest.raises(AttributeError):
        q.n = 3


def test_predictions():
    p = invop.predict_direct_costs(1, 1000)
    assert p.direct_products == pytest.approx(2500.0)
    assert p.direct_sums == pytest.approx(14200.0)
    with pytest.raises(ValueError):
        invop.predict_direct_costs(0, 10)
    with pytest.raises(ValueError):
        invop.CostPrediction(-1.0, 0.0, 0.0, 0.0)


def test_device_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    q = invop.QuantizedMatrix(n=2, scale_digits=1, mantissas=np.eye(2, dtype=np.int64))
    with pytest.raises(invop.InvopError):
        invop.build_plan(q).planned_additions


def test_builder_loads_without_the_library(tmp_path):
    """__graft_entry__.build() must work on a fresh checkout, where importing
    the package fails because the library is not built yet: the builder
    module loads standalone."""
    import subprocess
    import sys

    code = ("import sys, __graft_entry__ as g; b = g._builder(); "
            "assert 'paper_1602_00001_b200' not in sys.modules; "
            "assert b.LIB.name == 'libinvop_b200.so' and b.sources(); print('ok')")
    out = subprocess.run([sys.executable, "-c", code], cwd=str(_lib.LIB_PATH.parent.parent),
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr
