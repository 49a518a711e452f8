#!/bin/bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored; it
# travels to the GPU box with the gpurun snapshot) together with its own test
# files (baseline/_ref/ref_tests), which tests/test_ref_suite.py runs against
# this build through the sys.modules alias.  /root/reference is read-only, so
# the build happens from a scratch copy.
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "no reference at $SRC"; exit 0; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
mkdir -p "$REPO/baseline/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$REPO/baseline/_ref" "$TMP/pkg"
mkdir -p "$REPO/baseline/_ref/ref_tests"
cp "$SRC"/tests/*.py "$REPO/baseline/_ref/ref_tests/"
rm -rf "$TMP"
ls "$REPO/baseline/_ref"
