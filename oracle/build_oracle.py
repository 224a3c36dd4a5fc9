"""TEST INFRASTRUCTURE — build recipe for the oracle (checker only).

1. oracle/liboracle.so  — our C restatement (apply_ref.c), gcc -O3
   -ffp-contract=off like the reference's own build (pkg/setup.py:11-13).
2. oracle/_ref/         — the reference's own compiled kernel: Cython
   translates /root/reference/pkg/src/invop/_kernels/_native.pyx (read where it
   lies, never copied into the repo) to C under oracle/_ref/build/, and gcc
   links oracle/_ref/_native<EXT_SUFFIX>. Only attempted when /root/reference
   exists (this container); the GPU box uses the prebuilt .so.
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_PYX = Path("/root/reference/pkg/src/invop/_kernels/_native.pyx")
REF_DIR = HERE / "_ref"
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"


def build_oracle() -> Path:
    out = HERE / "liboracle.so"
    src = HERE / "apply_ref.c"
    if out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    cmd = ["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-pthread", str(src), "-o", str(out)]
    subprocess.run(cmd, check=True)
    return out


def build_reference() -> Path | None:
    target = REF_DIR / ("_native" + EXT)
    if not REF_PYX.exists():
        return target if target.exists() else None
    if target.exists() and target.stat().st_mtime >= REF_PYX.stat().st_mtime:
        return target
    bdir = REF_DIR / "build"
    bdir.mkdir(parents=True, exist_ok=True)
    c_file = bdir / "_native.c"
    subprocess.run(
        [sys.executable, "-m", "cython", "-3", "--module-name", "_native", str(REF_PYX), "-o", str(c_file)],
        check=True,
    )
    inc = sysconfig.get_paths()["include"]
    cmd = ["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-I", inc, str(c_file), "-o", str(target)]
    subprocess.run(cmd, check=True)
    return target


def build_all() -> None:
    build_oracle()
    build_reference()


if __name__ == "__main__":
    build_all()
    print(HERE / "liboracle.so", REF_DIR)
