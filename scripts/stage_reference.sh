#!/bin/sh
# Install the unmodified reference into baseline/_ref (git-ignored, travels to
# the GPU box with gpurun) and stage its own test suite and shipped config
# next to it, so tests/test_gpu_refsuite.py can run the reference's tests
# against the GPU path there (/root/reference does not exist on the box).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC (run in the build container)"; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg" >/dev/null
rm -rf "$ROOT/baseline/_ref/pkg"
mkdir -p "$ROOT/baseline/_ref/pkg"
cp -r "$SRC/tests" "$SRC/configs" "$ROOT/baseline/_ref/pkg/"
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref, suite staged in $ROOT/baseline/_ref/pkg/tests"
