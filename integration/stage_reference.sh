#!/bin/bash
# Stage the unmodified reference for the GPU box (run in the build container,
# where /root/reference exists).  baseline/_ref is git-ignored but NOT
# gpurun-ignored, so it travels with the repo snapshot:
#   baseline/_ref/spelunk   the package (the one offline pip install the task allows)
#   baseline/_ref/tests     the reference's own test suite, run through the
#                           Option-B shim by tests/test_gpu_reference_suite.py
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${1:-/root/reference}"
TMP="$(mktemp -d)"
cp -r "$REF/pkg" "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref/tests"
cp -r "$REF/pkg/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
echo "staged reference into $ROOT/baseline/_ref"
