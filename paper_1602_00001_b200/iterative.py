"""Cost-model formulas of the iterative baseline (paper Eqs. 7-8).

Only the two prediction formulas that `predict_direct_costs` reports beside
the direct method are kept (reference iterative.py:84-96). The SOR /
Gauss-Seidel solvers themselves are the comparison baseline of the paper, not
the inverse apply, and are out of scope.
"""

from __future__ import annotations

import math

LN10 = math.log(10.0)


def predict_iterations(n_total: int, digits: int) -> float:
    """Iteration-count model (2 ln 10 / pi) * m * N."""
    if n_total < 1:
        raise ValueError("n_total must be at least 1")
    if digits < 0:
        raise ValueError("digits must be non-negative")
    return (2.0 * LN10 / math.pi) * digits * n_total


def predict_iterative_total(n_total: int, digits: int) -> float:
    """Total-cost model 5N per sweep times the predicted iterations."""
    return 5.0 * n_total * predict_iterations(n_total, digits)
