#!/usr/bin/env bash
# Install the UNMODIFIED reference package (sparsekv, pure Python) into
# baseline/_ref for the bench's reference arm, and copy its own test suite
# next to it for tests/test_gpu_reference_suite.py (the drop-in check).
# baseline/_ref is git-ignored (not product source) but NOT gpurun-ignored,
# so it travels to the GPU box, where /root/reference does not exist.
# The reference tree is read-only: build from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${1:-/root/reference}"
DEST="$ROOT/baseline/_ref"
rm -rf /tmp/sparsekv_src && cp -r "$REF/pkg" /tmp/sparsekv_src
rm -rf "$DEST" && mkdir -p "$DEST"
# matplotlib (needed only by the reference's report plots) is not in the
# offline wheelhouse: --no-deps, numpy is already in the image
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DEST" /tmp/sparsekv_src
cp -r "$REF/pkg/tests" "$DEST/sparsekv_tests"
echo "installed sparsekv into $DEST (tests in $DEST/sparsekv_tests)"
