"""Shared test setup.

Markers: `gpu` — needs a CUDA device (run with -m gpu on the B200 box).
Everything unmarked runs on CPU: the oracle against golden vectors, host
logic, and that the C-ABI library loads and exports its header's symbols.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / (name + ".npz")))
        return cache[name]

    return load


def random_quantized_mant(rng, n, digits):
    """The reference's conftest generator (pkg/tests/conftest.py:33-38)."""
    pool = rng.integers(1, 10 ** (digits + 1) + 9, size=int(rng.integers(1, 5)))
    mant = rng.choice(pool, size=(n, n)) * rng.choice([-1, 0, 1], size=(n, n))
    return mant.astype(np.int64)


def battery_cases(g):
    meta = g["meta"]
    mo = xo = 0
    for n, m, mults, adds in meta:
        n = int(n)
        yield (int(n), int(m), g["mant"][mo:mo + n * n].reshape(n, n), g["x"][xo:xo + n],
               g["y"][xo:xo + n], (int(mults), int(adds)))
        mo += n * n
        xo += n
