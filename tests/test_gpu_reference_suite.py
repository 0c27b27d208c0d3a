"""The reference's OWN tests, run against the B200 library through the
Option-B drop-in (integration/_b200.py).

The unmodified reference package and its test suite are staged into
baseline/_ref by integration/stage_reference.sh (git-ignored, travels to the
GPU box).  The test copies the package to a temp dir, installs the shim
(range_bound_batch / interval_forward_batch dispatch to the C-ABI when
SPELUNK_BACKEND=b200, FP64 kernels) and runs, in a subprocess:

  test_range_core.py   incl. test_batch_matches_single_composition (:286-304,
                       abs 1e-12 against the single-form composition)
  test_rays.py         incl. the step-safety spy (:177-201, which wraps the
                       dispatched range_bound_batch) and threads=4 parity
                       (:146-150: concurrent callers of the host entry point)
  test_spatial.py::TestBuildSpatialTree (:61-127)
  test_meshing.py      (:63-106)

and asserts they pass and that the GPU path really ran (call counter written
by the shim at exit).
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
LIB = ROOT / "paper_2202_02444_b200" / "_spk.so"
sys.path.insert(0, str(ROOT / "integration"))

pytestmark = pytest.mark.gpu

SUITE = [
    "tests/test_range_core.py",
    "tests/test_rays.py",
    "tests/test_spatial.py::TestBuildSpatialTree",
    "tests/test_meshing.py",
]


@pytest.mark.skipif(not (REF / "spelunk").is_dir() or not (REF / "tests").is_dir(),
                    reason="reference not staged (run integration/stage_reference.sh in the build container)")
def test_reference_suite_through_shim(tmp_path):
    import shutil

    from install_shim import install

    install(REF / "spelunk", tmp_path / "pkg")
    shutil.copytree(REF / "tests", tmp_path / "tests", ignore=shutil.ignore_patterns("__pycache__"))
    calls = tmp_path / "calls.txt"
    env = dict(os.environ, PYTHONPATH=str(tmp_path / "pkg"), SPELUNK_BACKEND="b200", SPELUNK_B200_LIB=str(LIB),
               SPELUNK_B200_CALLS=str(calls), SPELUNK_B200_PRECISION="fp64", PYTHONDONTWRITEBYTECODE="1")
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *SUITE],
                         cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1200)
    print(res.stdout[-4000:])
    print(res.stderr[-2000:])
    assert res.returncode == 0, res.stdout[-4000:]
    n = int(calls.read_text())
    print(f"reference suite: {n} range_bound_batch calls served by the B200 library")
    assert n > 100


# FP32 arithmetic cannot meet these exact-value assertions (1e-12 composition,
# exact linear / identity ranges, [-3, 3] dependency bound, exact full-vs-
# condensed ordering); everything else of the suite holds in FP32 too
FP32_EXACT_ONLY = [
    "tests/test_range_core.py::TestIntervalForward::test_dependency_problem_bound",
    "tests/test_range_core.py::TestIntervalForward::test_identity",
    "tests/test_range_core.py::TestRangeBound::test_batch_matches_single_composition",
    "tests/test_range_core.py::TestConservatism::test_full_tighter_than_condensed",
    "tests/test_range_core.py::TestAffineExactness::test_linear_networks_are_exact",
]


@pytest.mark.skipif(not (REF / "spelunk").is_dir() or not (REF / "tests").is_dir(),
                    reason="reference not staged (run integration/stage_reference.sh in the build container)")
def test_reference_suite_through_shim_fp32_refine(tmp_path):
    """The same suite with SPELUNK_B200_PRECISION=fp32-refine (FP32 kernels,
    near-certifiable boxes re-bounded in FP64): every tree, ray (spy and
    threaded parity included), mesh and range test passes except the five
    exact-arithmetic assertions above."""
    import shutil

    from install_shim import install

    install(REF / "spelunk", tmp_path / "pkg")
    shutil.copytree(REF / "tests", tmp_path / "tests", ignore=shutil.ignore_patterns("__pycache__"))
    calls = tmp_path / "calls.txt"
    env = dict(os.environ, PYTHONPATH=str(tmp_path / "pkg"), SPELUNK_BACKEND="b200", SPELUNK_B200_LIB=str(LIB),
               SPELUNK_B200_CALLS=str(calls), SPELUNK_B200_PRECISION="fp32-refine", PYTHONDONTWRITEBYTECODE="1")
    deselect = [a for t in FP32_EXACT_ONLY for a in ("--deselect", t)]
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *SUITE, *deselect],
                         cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1200)
    print(res.stdout[-3000:])
    assert res.returncode == 0, res.stdout[-4000:]
    assert "75 passed" in res.stdout
    assert int(calls.read_text()) > 100
