#!/usr/bin/env bash
# Install the UNMODIFIED reference (cutdg) into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot), the one offline install
# the task allows.  /root/reference is read-only and has no top-level
# pyproject (the package lives in pkg/), so it is built from a copy under /tmp;
# --no-deps: numpy/scipy are already in the image.  The reference's own test
# files are placed next to it (baseline/_ref/cutdg_tests) so that
# tests/test_reference_suite_gpu.py can run their bodies against this package
# on the GPU box, where /root/reference does not exist.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference}"
TMP="$(mktemp -d /tmp/cutdg_src.XXXXXX)"
cp -r "$SRC/pkg/." "$TMP/"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" "$TMP"
mkdir -p "$ROOT/baseline/_ref/cutdg_tests"
cp "$SRC"/pkg/tests/test_*.py "$ROOT/baseline/_ref/cutdg_tests/"
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
