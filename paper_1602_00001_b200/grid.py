"""Grid geometry and 5-point operators (setup input of the apply path).

Dense API parity with /root/reference/pkg/src/invop/grid.py (Grid2D :26-79,
OperatorMatrix :87-107, build_uniform :157-169, build_variable :172-186,
assemble_rhs :189-198, MAX_DENSE_N :21). Every operator built here also
carries its five stencil diagonals (`StencilOperator`), which is the form the
device constructor of L^-1 consumes (csrc/construct.cu): a 5-point operator is
block tridiagonal over grid lines, so its inverse rows come from block solves
instead of a dense O(N^3) LU, and never need the N x N dense matrix.

Two interior-only operators used by the benchmark configurations are defined
here as well (BASELINE.json configs):
  * uniform_interior(n): unit-diagonal Poisson operator on the n x n interior
    points, Dirichlet-0 neighbours dropped — the interior block of the
    reference's full-grid build_uniform (its inverse equals the interior block
    of the reference's full inverse);
  * variable_interior(n, seed): the variable-permittivity, non-uniform-spacing
    operator of config 4 (definition pinned in DESIGN.md).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Union

import numpy as np

from .errors import CapacityError

MAX_DENSE_N = 8192

FieldSpec = Optional[Union[Callable, np.ndarray, list, tuple]]


@dataclass(frozen=True)
class Grid2D:
    """Uniform rectangular lattice on [0, length]^2, points p = (i-1)*nx + (j-1)."""

    nx: int
    ny: int
    length: float = 1.0

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2:
            raise ValueError("grid needs at least 2 points per axis, got (%d, %d)" % (self.nx, self.ny))
        if not (self.length > 0.0 and np.isfinite(self.length)):
            raise ValueError("domain length must be positive and finite")

    @property
    def n(self) -> int:
        return self.nx * self.ny

    @property
    def hx(self) -> float:
        return self.length / (self.nx - 1)

    @property
    def hy(self) -> float:
        return self.length / (self.ny - 1)

    def index(self, i: int, j: int) -> int:
        if not (1 <= i <= self.ny and 1 <= j <= self.nx):
            raise ValueError("point (%d, %d) outside grid (%d, %d)" % (i, j, self.nx, self.ny))
        return (i - 1) * self.nx + (j - 1)

    def coords(self, p: int) -> tuple:
        if not 0 <= p < self.n:
            raise ValueError("point index %d outside 0..%d" % (p, self.n - 1))
        i, j = divmod(p, self.nx)
        return self.hx * j, self.hy * i

    def boundary_mask(self) -> np.ndarray:
        i, j = np.divmod(np.arange(self.n), self.nx)
        return (i == 0) | (i == self.ny - 1) | (j == 0) | (j == self.nx - 1)

    def interior_mask(self) -> np.ndarray:
        return ~self.boundary_mask()

    def sample(self, fn: Callable) -> np.ndarray:
        out = np.empty(self.n, dtype=np.float64)
        for p in range(self.n):
            x, y = self.coords(p)
            out[p] = fn(x, y)
        return out


@dataclass(frozen=True)
class StencilOperator:
    """5-point operator on an nx x ny lattice of unknowns p = r*nx + c.

    Row p: diag[p] on the diagonal, -w_west[p] at (r, c-1), -w_east[p] at
    (r, c+1), -w_south[p] at (r-1, c), -w_north[p] at (r+1, c). Couplings that
    would leave the lattice must be zero.
    """

    nx: int
    ny: int
    diag: np.ndarray
    w_west: np.ndarray
    w_east: np.ndarray
    w_south: np.ndarray
    w_north: np.ndarray

    def __post_init__(self):
        n = self.nx * self.ny
        for name in ("diag", "w_west", "w_east", "w_south", "w_north"):
            arr = np.ascontiguousarray(getattr(self, name), dtype=np.float64)
            if arr.shape != (n,):
                raise ValueError("%s must have length nx*ny=%d" % (name, n))
            if not np.isfinite(arr).all():
                raise ValueError("%s must be finite" % name)
            arr.setflags(write=False)
            object.__setattr__(self, name, arr)
        r, c = np.divmod(np.arange(n), self.nx)
        if (np.any(self.w_west[c == 0] != 0) or np.any(self.w_east[c == self.nx - 1] != 0)
                or np.any(self.w_south[r == 0] != 0) or np.any(self.w_north[r == self.ny - 1] != 0)):
            raise ValueError("stencil couples to a point outside the lattice")

    @property
    def n(self) -> int:
        return self.nx * self.ny

    def to_dense(self) -> np.ndarray:
        n, nx = self.n, self.nx
        if n > MAX_DENSE_N:
            raise CapacityError("dense operator with N=%d > limit %d" % (n, MAX_DENSE_N))
        a = np.zeros((n, n), dtype=np.float64)
        p = np.arange(n)
        a[p, p] = self.diag
        for w, off in ((self.w_west, -1), (self.w_east, 1), (self.w_south, -nx), (self.w_north, nx)):
            m = w != 0
            a[p[m], p[m] + off] = -w[m]
        return a

    def to_sparse(self):
        """scipy.sparse CSR form (used by tests and the oracle only)."""
        import scipy.sparse as sp

        n, nx = self.n, self.nx
        p = np.arange(n)
        rows, cols, vals = [p], [p], [self.diag]
        for w, off in ((self.w_west, -1), (self.w_east, 1), (self.w_south, -nx), (self.w_north, nx)):
            m = w != 0
            rows.append(p[m]); cols.append(p[m] + off); vals.append(-w[m])
        return sp.csr_matrix(
            (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)
        )


def _freeze(arr: np.ndarray) -> np.ndarray:
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class OperatorMatrix:
    """Dense N x N system matrix with boundary-identity rows (reference
    grid.py:87-107). `stencil` holds the same operator as 5-point diagonals."""

    n: int
    entries: np.ndarray
    is_boundary: np.ndarray
    stencil: Optional[StencilOperator] = None

    def __post_init__(self):
        ent = np.ascontiguousarray(self.entries, dtype=np.float64)
        tags = np.ascontiguousarray(self.is_boundary, dtype=np.bool_)
        if ent.shape != (self.n, self.n):
            raise ValueError("entries shape %s does not match n=%d" % (ent.shape, self.n))
        if tags.shape != (self.n,):
            raise ValueError("row tag vector must have length n")
        object.__setattr__(self, "entries", _freeze(ent))
        object.__setattr__(self, "is_boundary", _freeze(tags))


@dataclass(frozen=True)
class CoefficientField:
    beta: np.ndarray

    def __post_init__(self):
        b = np.ascontiguousarray(self.beta, dtype=np.float64)
        if b.ndim != 1:
            raise ValueError("beta must be a flat per-point vector")
        if not np.isfinite(b).all():
            raise ValueError("beta values must be finite")
        object.__setattr__(self, "beta", _freeze(b))


@dataclass(frozen=True)
class SourceField:
    f: FieldSpec
    g: FieldSpec = None


def _point_values(grid: Grid2D, spec, what: str) -> np.ndarray:
    if spec is None:
        return np.zeros(grid.n, dtype=np.float64)
    if callable(spec):
        return grid.sample(spec)
    vals = np.ascontiguousarray(spec, dtype=np.float64)
    if vals.shape != (grid.n,):
        raise ValueError("%s samples must have length %d, got shape %s" % (what, grid.n, vals.shape))
    return vals


def _check_capacity(grid: Grid2D) -> None:
    if grid.n > MAX_DENSE_N:
        raise CapacityError(
            "dense operator for %dx%d grid needs N=%d > limit %d"
            % (grid.nx, grid.ny, grid.n, MAX_DENSE_N)
        )


def _full_grid_stencil(grid: Grid2D, beta: Optional[np.ndarray]) -> StencilOperator:
    n, nx = grid.n, grid.nx
    mask = grid.boundary_mask()
    interior = ~mask
    p = np.arange(n)
    ws = {}
    for name, off in (("w_west", -1), ("w_east", 1), ("w_south", -nx), ("w_north", nx)):
        w = np.zeros(n)
        q = p[interior] + off
        w[interior] = 0.25 * (beta[q] if beta is not None else 1.0)
        ws[name] = w
    return StencilOperator(nx=grid.nx, ny=grid.ny, diag=np.ones(n), **ws)


def build_uniform(grid: Grid2D) -> OperatorMatrix:
    """u - 0.25*(sum of neighbours) on interior rows, identity on boundary rows
    (reference grid.py:157-169)."""
    _check_capacity(grid)
    st = _full_grid_stencil(grid, None)
    return OperatorMatrix(n=grid.n, entries=st.to_dense(), is_boundary=grid.boundary_mask(), stencil=st)


def build_variable(grid: Grid2D, coeffs: CoefficientField) -> OperatorMatrix:
    """Interior rows take -0.25*beta[q] at neighbour q (reference grid.py:172-186)."""
    _check_capacity(grid)
    if coeffs.beta.shape != (grid.n,):
        raise ValueError("coefficient field has %d values, grid has %d points" % (coeffs.beta.size, grid.n))
    st = _full_grid_stencil(grid, coeffs.beta)
    return OperatorMatrix(n=grid.n, entries=st.to_dense(), is_boundary=grid.boundary_mask(), stencil=st)


def assemble_rhs(grid: Grid2D, source: SourceField) -> np.ndarray:
    """g at boundary slots, -f*hx*hy/4 at interior slots (reference grid.py:189-198)."""
    mask = grid.boundary_mask()
    fv = _point_values(grid, source.f, "source")
    gv = _point_values(grid, source.g, "boundary")
    rhs = np.empty(grid.n, dtype=np.float64)
    rhs[mask] = gv[mask]
    rhs[~mask] = -fv[~mask] * (grid.hx * grid.hy / 4.0)
    return rhs


def analytic_solution(x: float, y: float) -> float:
    return (x ** 4 - x ** 3) * (y ** 3 - y ** 2)


def test_source(x: float, y: float) -> float:
    return (12.0 * x ** 2 - 6.0 * x) * (y ** 3 - y ** 2) + (x ** 4 - x ** 3) * (6.0 * y - 2.0)


test_source.__test__ = False  # not a pytest test


# ---------------------------------------------------------------- interior operators
def uniform_interior(n: int, ny: Optional[int] = None) -> StencilOperator:
    """Unit-diagonal 5-point Poisson operator on n x ny interior points."""
    ny = n if ny is None else ny
    if n < 1 or ny < 1:
        raise ValueError("need at least one interior point")
    N = n * ny
    r, c = np.divmod(np.arange(N), n)
    q = 0.25
    return StencilOperator(
        nx=n, ny=ny, diag=np.ones(N),
        w_west=np.where(c > 0, q, 0.0), w_east=np.where(c < n - 1, q, 0.0),
        w_south=np.where(r > 0, q, 0.0), w_north=np.where(r < ny - 1, q, 0.0),
    )


def nonuniform_spacing(n: int) -> np.ndarray:
    """n+1 interval widths h_i ∝ 1 + 0.3 sin(2π i / n), i = 0..n, summing to 1."""
    i = np.arange(n + 1)
    h = 1.0 + 0.3 * np.sin(2.0 * np.pi * i / n)
    return h / h.sum()


def smoothed_permittivity(n: int, seed: int) -> np.ndarray:
    """(n+2)^2 node permittivities: lognormal(0, 0.5) from default_rng(seed),
    then a 5-point box mean with edge padding."""
    rng = np.random.default_rng(seed)
    eps = rng.lognormal(mean=0.0, sigma=0.5, size=(n + 2, n + 2))
    pad = np.pad(eps, 1, mode="edge")
    return (pad[1:-1, 1:-1] + pad[:-2, 1:-1] + pad[2:, 1:-1] + pad[1:-1, :-2] + pad[1:-1, 2:]) / 5.0


def variable_interior(n: int, seed: int = 104) -> StencilOperator:
    """Config-4 operator: -d/dx(eps du/dx) - d/dy(eps du/dy) on a non-uniform
    (n+2) x (n+2) node grid, Dirichlet-0 boundary, n x n interior unknowns.

    Face permittivity is the harmonic mean of the two nodes; the weight of a
    neighbour across face f is eps_f / (h_f * Delta), Delta the half-sum of the
    two intervals adjacent to the node; rows are scaled to unit diagonal and
    couplings to boundary nodes are dropped.
    """
    h = nonuniform_spacing(n)          # intervals between nodes 0..n+1
    eps = smoothed_permittivity(n, seed)  # [row node][col node]
    N = n * n
    r, c = np.divmod(np.arange(N), n)
    R, Cc = r + 1, c + 1                # node indices of the unknowns
    e0 = eps[R, Cc]

    def hmean(a, b):
        return 2.0 * a * b / (a + b)

    dx = 0.5 * (h[Cc - 1] + h[Cc])
    dy = 0.5 * (h[R - 1] + h[R])
    w_w = hmean(e0, eps[R, Cc - 1]) / (h[Cc - 1] * dx)
    w_e = hmean(e0, eps[R, Cc + 1]) / (h[Cc] * dx)
    w_s = hmean(e0, eps[R - 1, Cc]) / (h[R - 1] * dy)
    w_n = hmean(e0, eps[R + 1, Cc]) / (h[R] * dy)
    d = w_w + w_e + w_s + w_n
    return StencilOperator(
        nx=n, ny=n, diag=np.ones(N),
        w_west=np.where(c > 0, w_w / d, 0.0), w_east=np.where(c < n - 1, w_e / d, 0.0),
        w_south=np.where(r > 0, w_s / d, 0.0), w_north=np.where(r < n - 1, w_n / d, 0.0),
    )
