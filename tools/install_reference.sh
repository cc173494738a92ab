#!/usr/bin/env bash
# Offline install of the reference package (rhymesim) into baseline/_ref (git-ignored; it travels to the
# GPU box with the gpurun snapshot).  The reference's own tests are copied beside it so the drop-in can
# be run against them on the box, where /root/reference does not exist (tests/test_reference_suite_gpu.py).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${REF:-/root/reference}"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$REF/pkg"
rm -rf "$ROOT/baseline/_ref/rhymesim_tests"
cp -r "$REF/pkg/tests" "$ROOT/baseline/_ref/rhymesim_tests"
echo "installed rhymesim + tests into $ROOT/baseline/_ref"
