#!/bin/sh
# Copy the reference's own Python smoke test (proj/python/tests/test_smoke.py)
# into tests/_ref/ (git-ignored, so it is not part of this repository's
# history, but it travels to the GPU box with the gpurun snapshot), where
# tests/test_gpu_ref_smoke.py runs it UNCHANGED against this repository's
# pyising. Run in the container that has /root/reference (build() does).
set -e
REF=${REF:-/root/reference/proj/python/tests/test_smoke.py}
DEST=$(dirname "$0")/../tests/_ref
[ -f "$REF" ] || { echo "no $REF: skipped"; exit 0; }
mkdir -p "$DEST"
# (named ref_*.py: collected only when run explicitly, with pyising on the path)
cp "$REF" "$DEST/ref_test_smoke.py"
echo "vendored $REF -> $DEST/ref_test_smoke.py"
