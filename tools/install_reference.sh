#!/usr/bin/env bash
# Install the UNMODIFIED reference package (axlandau, /root/reference/pkg) into
# baseline/_ref (git-ignored, travels to the GPU box with the gpurun snapshot),
# plus its own test suite under baseline/_ref/axlandau_tests, so the GPU box --
# where /root/reference does not exist -- can run the reference's tests with
# the B200 path installed (tests/test_gpu_reference_suite.py).  Offline: the
# wheelhouse only; numpy/scipy/numba are already in the image.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"          # the build writes egg-info into the source tree
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/axlandau_tests"
cp "$SRC/test_output.txt" "$ROOT/baseline/_ref/axlandau_tests/" 2>/dev/null || true
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref"
