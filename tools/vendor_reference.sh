#!/bin/bash
# Installs the UNMODIFIED reference package (wordsort) into baseline/_ref and
# copies its test modules next to it (baseline/_ref/ref_tests). Both paths are
# git-ignored but travel to the GPU box with the gpurun snapshot, where
# /root/reference does not exist. Run here (the reference is read-only, so the
# build works on a copy under /tmp).
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { cat "$TMP/pip.log"; exit 1; }
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
mkdir -p "$ROOT/baseline/_ref/data" && cp -r "$SRC/data/." "$ROOT/baseline/_ref/data/"
rm -rf "$TMP"
echo "reference installed: $(ls "$ROOT/baseline/_ref")"
