"""The five BASELINE.json workloads as seeded synthetic inputs.

There is no public dataset: BASELINE.json specifies synthetic operators and
right-hand sides; the seeds and the config-4 operator definition are pinned
here and recorded in DESIGN.md.

  cfg 1  uniform 10x10 interior (N=100),     m=3, 1 RHS  rng(101) N(0,1),        fp64 (bitwise)
  cfg 2  uniform 50x50 interior (N=2500),    m=4, 16 RHS rng(102) N(0,1),        fp32
  cfg 3  uniform 100x100 interior (N=1e4),   m=4, 1 RHS  8 Gaussian blobs rng(103), fp32
  cfg 4  variable eps, non-uniform 128x128 (N=16384), m=5, 1 RHS rng(1041) N(0,1), fp32
  cfg 5  uniform 256x256 interior (N=65536), m=4, 64 RHS rng(105) N(0,1)+moving blob, fp32

"k significant digits" of BASELINE.json is read as the reference's only
quantization mode, k decimal places (quant.py:48-65); see DESIGN.md.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .grid import StencilOperator, uniform_interior, variable_interior


@dataclass(frozen=True)
class Config:
    key: int
    name: str
    n: int             # interior points per side
    digits: int
    nrhs: int
    precision: str     # "f64" (bitwise ordered) or "f32"
    operator: Callable[[], StencilOperator]
    rhs: Callable[[], np.ndarray]   # [nrhs, N] float64

    @property
    def N(self) -> int:
        return self.n * self.n


def _gaussian_blobs(n: int, seed: int, count: int = 8) -> np.ndarray:
    rng = np.random.default_rng(seed)
    centers = rng.uniform(0.0, 1.0, size=(count, 2))
    amps = rng.uniform(-1.0, 1.0, size=count)
    h = 1.0 / (n + 1)
    sigma = 5.0 * h
    coord = np.arange(1, n + 1) * h
    yy, xx = np.meshgrid(coord, coord, indexing="ij")   # row r = y (slow), col c = x
    rho = np.zeros((n, n))
    for (cx, cy), a in zip(centers, amps):
        rho += a * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2.0 * sigma ** 2))
    return rho.reshape(1, -1)


def _moving_blob_batch(n: int, seed: int, k: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal((k, n * n))
    h = 1.0 / (n + 1)
    sigma = 5.0 * h
    coord = np.arange(1, n + 1) * h
    yy, xx = np.meshgrid(coord, coord, indexing="ij")
    for t in range(k):
        cx = 0.25 + 0.5 * t / max(k - 1, 1)
        noise[t] += np.exp(-((xx - cx) ** 2 + (yy - 0.5) ** 2) / (2.0 * sigma ** 2)).ravel()
    return noise


CONFIGS = {
    1: Config(1, "poisson-uniform-10x10-m3", 10, 3, 1, "f64",
              lambda: uniform_interior(10),
              lambda: np.random.default_rng(101).standard_normal((1, 100))),
    2: Config(2, "poisson-uniform-50x50-m4", 50, 4, 16, "f32",
              lambda: uniform_interior(50),
              lambda: np.random.default_rng(102).standard_normal((16, 2500))),
    3: Config(3, "poisson-uniform-100x100-m4", 100, 4, 1, "f32",
              lambda: uniform_interior(100),
              lambda: _gaussian_blobs(100, 103)),
    4: Config(4, "variable-eps-nonuniform-128x128-m5", 128, 5, 1, "f32",
              lambda: variable_interior(128, seed=104),
              lambda: np.random.default_rng(1041).standard_normal((1, 16384))),
    5: Config(5, "poisson-uniform-256x256-m4-batch64", 256, 4, 64, "f32",
              lambda: uniform_interior(256),
              lambda: _moving_blob_batch(256, 105, 64)),
}


def get(key: int) -> Config:
    return CONFIGS[int(key)]
