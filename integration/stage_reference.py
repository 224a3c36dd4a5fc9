"""Stage a COPY of the reference package with the b200 backend wired in.

    python integration/stage_reference.py        # -> baseline/_ref/pkg

What a maintainer of the reference would do to adopt the drop-in, applied to
a copy (never to /root/reference, which is read-only):

1. copy /root/reference/pkg to baseline/_ref/pkg (git-ignored; it travels to
   the GPU box with the gpurun snapshot, /root/reference does not);
2. `integration/enable_b200.py`: add the `b200` branch to the backend
   selection (`pkg/src/invop/_kernels/__init__.py:14-34`) and drop in
   `_kernels/_b200.py`;
3. put the reference's own compiled kernel next to it (`_native`, built by
   oracle/build_oracle.py from `_native.pyx` where it lies), so the staged
   package has all three backends — python, native, b200 — and the
   byte-equality tests can compare them;
4. copy `integration/test_b200_backend.py` into the staged tests directory.

tests/test_reference_suite.py (-m gpu) then runs the reference's own test
files with INVOP_BACKEND=b200 against this copy. Only done when
/root/reference exists (this container); on the GPU box the staged copy is
used as shipped.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
REF_PKG = Path("/root/reference/pkg")
STAGE = ROOT / "baseline" / "_ref" / "pkg"


def _ignore(_dir, names):
    return [n for n in names if n in ("build", "__pycache__", ".pytest_cache") or n.endswith(".so")
            or n.endswith(".egg-info")]


def stage(dest: Path = STAGE) -> Path | None:
    if not REF_PKG.exists():
        return dest if dest.exists() else None
    sys.path.insert(0, str(ROOT))
    from integration.enable_b200 import enable
    from oracle import build_oracle

    if dest.exists():
        shutil.rmtree(dest)
    dest.parent.mkdir(parents=True, exist_ok=True)
    shutil.copytree(REF_PKG, dest, ignore=_ignore)
    for p in dest.rglob("*"):
        p.chmod(p.stat().st_mode | 0o200)          # the source tree is read-only
    enable(dest)
    native = build_oracle.build_reference()
    if native is not None and native.exists():
        shutil.copyfile(native, dest / "src" / "invop" / "_kernels" / native.name)
    shutil.copyfile(HERE / "test_b200_backend.py", dest / "tests" / "test_b200_backend.py")
    return dest


if __name__ == "__main__":
    print(stage())
