"""The reference's OWN test suite run against the drop-in backend.

integration/stage_reference.py (run by __graft_entry__.build()) stages a copy
of the reference package in baseline/_ref/pkg with the `b200` backend wired
into its kernel seam (`pkg/src/invop/_kernels/__init__.py:14-39`) — the change
INTEGRATION.md §2 describes — plus integration/test_b200_backend.py, the
reference's backend byte-equality pattern (`pkg/tests/test_backends.py:25-87`)
applied to the device backend.

On a GPU the whole reference suite runs twice in subprocesses: with
INVOP_BACKEND=native (the reference as shipped) and INVOP_BACKEND=b200
(every `invop.apply`, `apply_naive_quantized`, `dense_matvec`, `run_table1`,
CLI apply ... on libinvop_b200.so). The b200 run must fail exactly the tests
the native run fails (the reference itself fails
test_criterion_5_scaling_separation, independent of the backend), and every
test of test_b200_backend.py must pass.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
STAGE = ROOT / "baseline" / "_ref" / "pkg"

needs_stage = pytest.mark.skipif(
    not (STAGE / "src" / "invop" / "_kernels" / "_b200.py").exists(),
    reason="reference copy not staged (integration/stage_reference.py needs /root/reference)")


def _env(backend: str) -> dict:
    env = dict(os.environ)
    env["INVOP_BACKEND"] = backend
    env["PYTHONPATH"] = str(STAGE / "src")
    env["INVOP_B200_LIB"] = str(ROOT / "paper_1602_00001_b200" / "libinvop_b200.so")
    return env


def _run_suite(backend: str, *extra: str):
    res = subprocess.run(
        [sys.executable, "-m", "pytest", "tests", "-q", "-p", "no:cacheprovider", "-rf", *extra],
        cwd=STAGE, env=_env(backend), capture_output=True, text=True, timeout=1500)
    failed = set(re.findall(r"^FAILED (\S+)", res.stdout, re.M))
    m = re.search(r"(\d+) passed", res.stdout)
    return res, failed, int(m.group(1)) if m else 0


@needs_stage
def test_staged_reference_selects_b200():
    """The seam picks the backend at import (no GPU needed to load the library)."""
    res = subprocess.run([sys.executable, "-c", "import invop; print(invop.BACKEND)"],
                         env=_env("b200"), capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    assert res.stdout.strip() == "b200"


@pytest.mark.gpu
@needs_stage
def test_reference_suite_on_b200_backend():
    ours = "tests/test_b200_backend.py"
    res_n, failed_n, passed_n = _run_suite("native", "--ignore", ours)
    res_b, failed_b, passed_b = _run_suite("b200")
    print(res_b.stdout[-3000:])
    assert passed_n > 100, res_n.stdout[-3000:] + res_n.stderr[-3000:]
    # every test of the backend byte-equality module passes on the device
    assert not any(f.startswith(ours) for f in failed_b), sorted(failed_b)
    # the reference's own tests: the same outcome as with its compiled kernel
    assert failed_b == failed_n, {"b200 only": sorted(failed_b - failed_n),
                                  "native only": sorted(failed_n - failed_b)}
    assert passed_b > passed_n
