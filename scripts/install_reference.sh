#!/usr/bin/env bash
# Install the UNMODIFIED reference package (shardsim) into baseline/_ref, the
# one offline install the task allows (git-ignored; it travels to the GPU box
# with the snapshot).  Used by bench.py --impl reference (the reference's own
# CPU DenseKet) and by tests/test_reference_suite.py, which runs the
# reference's own test files (copied here as test infrastructure, never into
# the repo history) against the device DenseKet.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"            # the reference tree is read-only; setuptools writes build files
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/shardsim_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/shardsim_tests/"
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
