#!/bin/bash
# The reference arm's one offline install: the UNMODIFIED reference package
# (isochr, pure Python + numba) into baseline/_ref (git-ignored; it travels to
# the GPU box with the repo snapshot), plus a copy of its own test suite for
# the kernel-seam run (tests/test_gpu_reference_suite.py).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference}
TMP=$(mktemp -d)
cp -r "$SRC/pkg" "$TMP/pkg"            # the build writes into the source tree
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" --upgrade
rm -rf "$ROOT/baseline/_ref/isochr_tests"
cp -r "$SRC/pkg/tests" "$ROOT/baseline/_ref/isochr_tests"
rm -rf "$TMP"
echo "installed isochr into $ROOT/baseline/_ref"
