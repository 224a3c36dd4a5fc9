"""Install the b200 backend into a COPY of the reference package.

    python integration/enable_b200.py <path to a copy of the reference's pkg/>

Copies integration/_b200.py to <pkg>/src/invop/_kernels/_b200.py and adds the
`b200` branch to the backend selection in <pkg>/src/invop/_kernels/__init__.py
(/root/reference/pkg/src/invop/_kernels/__init__.py:14-34) — the two-line
change a maintainer of the reference would make. Idempotent. Never touches
/root/reference itself.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

BRANCH = '''elif _requested == "b200":
    from . import _b200 as _impl

    BACKEND = "b200"
'''


def enable(pkg: Path) -> Path:
    pkg = Path(pkg).resolve()
    if str(pkg).startswith("/root/reference"):
        raise ValueError("refusing to modify the read-only reference; pass a copy")
    kern = pkg / "src" / "invop" / "_kernels"
    init = kern / "__init__.py"
    text = init.read_text()
    if "_b200" not in text:
        anchor = 'elif _requested == "":'
        if anchor not in text:
            raise RuntimeError("unexpected _kernels/__init__.py layout in %s" % init)
        text = text.replace(anchor, BRANCH + anchor, 1)
        text = text.replace("\"INVOP_BACKEND must be 'native' or 'python', got %r\"",
                            "\"INVOP_BACKEND must be 'native', 'python' or 'b200', got %r\"")
        init.write_text(text)
    shutil.copyfile(HERE / "_b200.py", kern / "_b200.py")
    return kern / "_b200.py"


if __name__ == "__main__":
    print(enable(Path(sys.argv[1])))
