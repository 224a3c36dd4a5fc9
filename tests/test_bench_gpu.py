"""bench.py on the GPU: the contract keys of the JSON line, and the N>1 step
(NCCL all-gather + unshard captured in a CUDA graph) exercised with a one-rank
process group (INVOP_BENCH_DIST1) — the code path the multi-GPU scaling runs
take, kept alive on one-GPU boxes."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
        "clocks")


def _bench(extra_env, *args):
    env = dict(os.environ)
    env.update(extra_env)
    env.setdefault("MASTER_ADDR", "127.0.0.1")
    res = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=900, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _bench({}, "--config", "2", "--steps", "4", "--warmup", "3", "--no-cpu-baseline")
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["value"] > 0
    assert d["config"]["N"] == 2500 and d["config"]["nrhs"] == 16
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] and r["achieved"] > 0 and r["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["fp32_vs_fp64_relerr"] <= 1e-5
    assert d["quantization_error"]["value"] < 1e-2


def test_bench_sharded_step_one_rank():
    d = _bench({"INVOP_BENCH_DIST1": "1", "MASTER_PORT": "29533"}, "--config", "2", "--steps", "4",
               "--warmup", "3", "--no-cpu-baseline", "--no-quant-error")
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["cuda_graph"] is True            # apply + all-gather + unshard replayed as one graph
    assert d["gpu_launches"] >= 4             # library kernels per replay x steps
    assert "all-gather" in d["e2e"]["path"]
    assert d["fp32_vs_fp64_relerr"] <= 1e-5
