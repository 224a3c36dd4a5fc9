"""Table-1 and scaling studies on the device path.

API parity with /root/reference/pkg/src/invop/bench.py: `relative_error`
(Eq. 6, :73-85), `ErrorRow` / `ScalingRow` / `ScalingReport`, `run_table1`
(:120-140), `run_scaling` (:143-194), `emit_csv` (:201-223). Every inverse,
quantization, plan and apply runs on the GPU; grids are built as 5-point
stencils, so sides far beyond the reference's dense limit (MAX_DENSE_N = 8192,
n <= 90) are reachable.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np

from .applyplan import ApplyPlan, apply, predict_direct_costs
from .dense import DeviceOperator
from .errors import DegenerateProblemError
from .grid import Grid2D, SourceField, _full_grid_stencil, analytic_solution, assemble_rhs, test_source
from .quant import QuantizedMatrix

SCALING_HEADER = (
    "n,N,m,n_mult,n_add,alpha_mult,alpha_add,naive_mult,naive_add,"
    "pred_prod_eq9,pred_sum_eq10,pred_iter_eq7,pred_iter_total_eq8"
)
TABLE_HEADER = "n,digits,error"


@dataclass(frozen=True)
class ErrorRow:
    n: int
    digits: Union[int, str]
    error: float

    def __post_init__(self):
        if self.error < 0:
            raise ValueError("relative error cannot be negative")


@dataclass(frozen=True)
class ScalingRow:
    n: int
    big_n: int
    m: int
    n_mult: int
    n_add: int
    alpha_mult: float
    alpha_add: float
    naive_mult: int
    naive_add: int
    pred_products: float
    pred_sums: float
    pred_iterations: float
    pred_iter_total: float


@dataclass(frozen=True)
class ScalingReport:
    rows: tuple
    slopes: dict


def relative_error(numerical, grid: Grid2D) -> float:
    """Max-norm error against the analytic solution, normalised by the
    largest analytic magnitude (Eq. 6)."""
    u_num = np.ascontiguousarray(numerical, dtype=np.float64)
    if u_num.shape != (grid.n,):
        raise ValueError("vector length %s does not match grid size %d" % (u_num.shape, grid.n))
    u_anal = grid.sample(analytic_solution)
    denom = float(np.abs(u_anal).max())
    if denom == 0.0:
        raise DegenerateProblemError(
            "analytic solution vanishes at every point of the %dx%d grid" % (grid.nx, grid.ny))
    return float(np.abs(u_num - u_anal).max() / denom)


def _norm_digits(d):
    if d is None or (isinstance(d, str) and d.lower() == "none"):
        return "none"
    return int(d)


class _Cell:
    """Device operator, its factorisation and the test right-hand side for one grid side."""

    def __init__(self, n: int):
        import torch

        self.grid = Grid2D(n, n)
        self.rhs = assemble_rhs(self.grid, SourceField(f=test_source))
        self.op = DeviceOperator(_full_grid_stencil(self.grid, None)).factor()
        self.rhs_dev = torch.tensor(self.rhs, device="cuda")

    def dense_apply(self):
        """Unrounded route: fp64 inverse rows times rhs, ascending columns (bitwise like
        the reference's apply_dense)."""
        import ctypes as C

        import torch

        from . import _device as dev
        from . import _lib as L

        inv = self.op.inverse_rows()
        y = torch.empty(self.grid.n, dtype=torch.float64, device="cuda")
        L.check(L.lib.invop_dense_matvec(L.ptr(inv), self.grid.n, self.grid.n, self.grid.n,
                                         L.ptr(self.rhs_dev), L.ptr(y), C.c_void_p(dev.stream_ptr())),
                "dense_matvec")
        N = self.grid.n
        return y.cpu().numpy(), (N * N, N * (N - 1))

    def plan(self, m: int) -> ApplyPlan:
        dplan = self.op.quantized_rows(m)
        q = QuantizedMatrix(n=self.grid.n, scale_digits=m, _dplan=dplan)
        return ApplyPlan(n=q.n, scale_digits=m, _dplan=dplan)


def run_table1(grid_sides, digit_list) -> list:
    """One ErrorRow per (digits, n), digits in caller order, sides within."""
    cells = {}
    rows = []
    for d in digit_list:
        digits = _norm_digits(d)
        for n in grid_sides:
            n = int(n)
            if n not in cells:
                cells[n] = _Cell(n)
            c = cells[n]
            if digits == "none":
                u, _ = c.dense_apply()
            else:
                u, _ = apply(c.plan(digits), c.rhs)
            rows.append(ErrorRow(n=n, digits=digits, error=relative_error(u, c.grid)))
    return rows


def run_scaling(grid_sides, digit_list) -> ScalingReport:
    """Fast-apply operation counts across grid sizes and digits, beside the
    dense counts and the paper's cost models; log-log slopes per m."""
    sides = sorted({int(n) for n in grid_sides})
    digits = sorted({int(m) for m in digit_list})
    if not sides or not digits:
        raise ValueError("need at least one grid side and one digit setting")
    for m in digits:
        if m < 1:
            raise ValueError("scaling study needs m >= 1, got %d" % m)
    rows = []
    for n in sides:
        c = _Cell(n)
        big_n = c.grid.n
        for m in digits:
            plan = c.plan(m)
            _, counters = apply(plan, c.rhs)
            pred = predict_direct_costs(m, big_n)
            rows.append(ScalingRow(
                n=n, big_n=big_n, m=m, n_mult=counters.multiplications, n_add=counters.additions,
                alpha_mult=counters.multiplications / big_n, alpha_add=counters.additions / big_n,
                naive_mult=big_n * big_n, naive_add=big_n * (big_n - 1),
                pred_products=pred.direct_products, pred_sums=pred.direct_sums,
                pred_iterations=pred.iterations, pred_iter_total=pred.iterative_total))
    rows.sort(key=lambda r: (r.n, r.m))
    slopes = {}
    for m in digits:
        sub = [r for r in rows if r.m == m]
        if len(sub) < 2:
            continue
        log_n = np.log([r.big_n for r in sub])
        slopes[m] = (float(np.polyfit(log_n, np.log([r.n_mult for r in sub]), 1)[0]),
                     float(np.polyfit(log_n, np.log([r.n_add for r in sub]), 1)[0]))
    return ScalingReport(rows=tuple(rows), slopes=slopes)


def emit_csv(report, path) -> None:
    """Write a report in the reference's pinned CSV schema (bench.py:201-223)."""
    if isinstance(report, ScalingReport):
        lines = [SCALING_HEADER]
        for r in report.rows:
            lines.append("%d,%d,%d,%d,%d,%r,%r,%d,%d,%r,%r,%r,%r" % (
                r.n, r.big_n, r.m, r.n_mult, r.n_add, r.alpha_mult, r.alpha_add, r.naive_mult,
                r.naive_add, r.pred_products, r.pred_sums, r.pred_iterations, r.pred_iter_total))
    elif isinstance(report, (list, tuple)) and all(isinstance(r, ErrorRow) for r in report):
        lines = [TABLE_HEADER] + ["%d,%s,%.6g" % (r.n, r.digits, r.error) for r in report]
    else:
        raise TypeError("unsupported report type: %r" % type(report).__name__)
    with open(path, "w", encoding="ascii", newline="\n") as fh:
        fh.write("\n".join(lines))
        fh.write("\n")
