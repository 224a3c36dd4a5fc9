"""paper_1602_00001_b200 — B200 (sm_100a) implementation of the quantized
inverse-operator apply of arXiv 1602.00001, behind the public API of the
reference package `invop` (/root/reference/pkg/src/invop/__init__.py:10-59).

    import paper_1602_00001_b200 as invop
    q = invop.quantize(invop.invert(op), digits)      # device construct + K1
    plan = invop.build_plan(q)                          # compressed device layout
    y, counters = invop.apply(plan, x)                  # K2, bitwise == reference
    y32, _ = invop.apply(plan, x, precision="f32")      # K2 fp32 I/O, exact integer sums

All arithmetic runs in libinvop_b200.so (CUDA, sm_100a) through a C ABI
(include/invop_b200.h); importing the package without the built library
raises, and device calls without a GPU raise — there is no CPU fallback.
"""

from ._lib import LIB_PATH as _LIB_PATH  # noqa: F401  (fails loudly if not built)
from .applyplan import (
    ApplyPlan,
    CostPrediction,
    apply,
    apply_many,
    apply_naive_quantized,
    build_plan,
    predict_direct_costs,
)
from .cache import CacheEntry, entry_for, read_matrix, read_vector, write_matrix, write_vector
from .counting import OpCounters
from .dense import PIVOT_RTOL, DenseMatrix, DeviceOperator, apply_dense, invert, residual_check
from .errors import (
    CacheError,
    CapacityError,
    DegenerateProblemError,
    InvopError,
    MantissaOverflowError,
    SingularMatrixError,
)
from .grid import (
    MAX_DENSE_N,
    CoefficientField,
    Grid2D,
    OperatorMatrix,
    SourceField,
    StencilOperator,
    analytic_solution,
    assemble_rhs,
    build_uniform,
    build_variable,
    test_source,
    uniform_interior,
    variable_interior,
)
from .harness import (
    ErrorRow,
    ScalingReport,
    ScalingRow,
    emit_csv,
    relative_error,
    run_scaling,
    run_table1,
)
from .iterative import predict_iterations, predict_iterative_total
from .quant import MANTISSA_LIMIT, QuantizedMatrix, dequantize, quantize, sparsity_stats

BACKEND = "cuda-sm100a"
__version__ = "0.1.0"


def quantized_inverse(stencil, digits: int, row0: int = 0, rows: int = None) -> QuantizedMatrix:
    """Rows of L^-1 of a 5-point operator, built and quantized on the device
    without materialising the fp64 inverse (setup; K4 fused with K1)."""
    dplan = DeviceOperator(stencil).factor().quantized_rows(digits, row0, rows)
    if dplan.rows != dplan.n:
        raise ValueError("quantized_inverse with a row range returns a shard; use "
                         "DeviceOperator.quantized_rows")
    return QuantizedMatrix(n=dplan.n, scale_digits=digits, _dplan=dplan)


__all__ = [
    "BACKEND", "ApplyPlan", "CacheEntry", "CacheError", "entry_for", "read_matrix", "read_vector",
    "write_matrix", "write_vector", "CapacityError", "CoefficientField", "CostPrediction",
    "DegenerateProblemError", "DenseMatrix", "DeviceOperator", "Grid2D", "InvopError",
    "MANTISSA_LIMIT", "MAX_DENSE_N", "MantissaOverflowError", "OpCounters", "OperatorMatrix",
    "PIVOT_RTOL", "QuantizedMatrix", "SingularMatrixError", "SourceField", "StencilOperator",
    "analytic_solution", "apply", "apply_dense", "apply_many", "apply_naive_quantized",
    "assemble_rhs", "build_plan", "build_uniform", "build_variable", "dequantize", "invert",
    "predict_direct_costs", "predict_iterations", "predict_iterative_total", "quantize",
    "quantized_inverse", "residual_check", "sparsity_stats", "test_source", "uniform_interior",
    "variable_interior", "ErrorRow", "ScalingReport", "ScalingRow", "emit_csv", "relative_error",
    "run_scaling", "run_table1",
]
