#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# travels to the GPU box with the snapshot), as the bench's reference arm and
# the drop-in suite test (tests/test_gpu_reference_suite.py) need it:
#   - the package itself: pip install --no-deps (numpy / scipy / OpenCV are
#     in the image; pip's resolver cannot see them from /opt/wheelhouse);
#   - the reference's own test directory next to it (egostereo_tests), so the
#     suite can run against the installed device path on the GPU box, where
#     /root/reference does not exist.
# The build writes into the source tree, so it runs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference}"
TMP="$(mktemp -d)"
cp -r "$SRC/pkg" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/pkg/tests" "$ROOT/baseline/_ref/egostereo_tests"
rm -rf "$TMP"
echo "installed $(ls "$ROOT/baseline/_ref")"
