"""bench.py --impl reference runs the reference's own compiled kernel
(oracle/_ref) without loading libinvop_b200.so, on the same config dict as
our arm (same workload_config)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not list((ROOT / "oracle" / "_ref").glob("_native*.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_is_clean():
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                          "--steps", "2", "--warmup", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference"
    assert line["b200_library_loaded"] is False
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["config"]["N"] == 100 and line["config"]["nrhs"] == 1
    assert line["value"] > 0
