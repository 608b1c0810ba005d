#!/usr/bin/env bash
# One-time offline install of the unmodified reference (pure Python) into
# baseline/_ref (git-ignored; it travels to the GPU box with gpurun), plus a
# copy of its own test suite in baseline/_ref/ref_tests so the -m gpu
# integration test can run the reference's tests through binding.install().
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"   # the build writes into the source tree; the reference is read-only
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref/ref_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
rm -rf "$TMP"
echo "installed submap_slam into $ROOT/baseline/_ref (+ ref_tests)"
