"""Install the Option-B drop-in into a COPY of the reference package.

    python integration/install_shim.py <reference spelunk package dir> <dest dir>

Copies the package to <dest>/spelunk, adds `_b200.py`, and appends to
`range_core.py` the dispatch a maintainer would add at the top of
range_bound_batch / interval_forward_batch (range_core.py:547, 625).  The
reference tree itself is never modified.  Used by
tests/test_gpu_reference_suite.py to run the reference's own tests with
SPELUNK_BACKEND=b200.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

DISPATCH = '''

# ---- B200 drop-in (INTEGRATION.md, Option B) ------------------------------
import os as _os

_numpy_range_bound_batch = range_bound_batch
_numpy_interval_forward_batch = interval_forward_batch


def range_bound_batch(net, centers, axes, policy):
    if _os.environ.get("SPELUNK_BACKEND") == "b200":
        from . import _b200
        return _b200.range_bound_batch(net, centers, axes, policy)
    return _numpy_range_bound_batch(net, centers, axes, policy)


def interval_forward_batch(net, centers, axes):
    if _os.environ.get("SPELUNK_BACKEND") == "b200":
        from . import _b200
        return _b200.interval_forward_batch(net, centers, axes)
    return _numpy_interval_forward_batch(net, centers, axes)
'''


def install(src_pkg: Path, dest: Path) -> Path:
    src_pkg, dest = Path(src_pkg), Path(dest)
    out = dest / "spelunk"
    if out.exists():
        shutil.rmtree(out)
    shutil.copytree(src_pkg, out, ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copyfile(HERE / "_b200.py", out / "_b200.py")
    rc = out / "range_core.py"
    rc.write_text(rc.read_text() + DISPATCH)
    return out


if __name__ == "__main__":
    print(install(Path(sys.argv[1]), Path(sys.argv[2])))
