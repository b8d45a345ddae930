#!/usr/bin/env bash
# Installs the UNMODIFIED reference (/root/reference/pkg) into baseline/_ref
# (pip --target, offline wheelhouse) and copies its tests next to it, for the
# drop-in test (tests/test_dropin_reference.py).  baseline/_ref is
# git-ignored but travels to the GPU box with gpurun.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"   # the build writes egg-info into the source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/ref_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/ref_tests/"
rm -rf "$TMP"
echo "installed splinecast into $ROOT/baseline/_ref"
