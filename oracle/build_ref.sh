#!/usr/bin/env bash
# Build the UNMODIFIED reference package (/root/reference/pkg) into
# oracle/_ref/ (git-ignored; travels to the GPU box with the snapshot).
# The build needs a writable tree, so it runs from a scratch copy; sources
# are never copied into this repository.  Test/bench infrastructure only.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then
  echo "reference not present at $SRC; keeping existing oracle/_ref" >&2
  exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
chmod -R u+w "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
# the reference's own test-suite travels with the build (git-ignored): the
# drop-in test runs it against the B200 plugin (tests/test_gpu_dropin.py)
cp -r "$TMP/pkg/tests" "$HERE/_ref/_reference_tests"
PYTHONPATH="$HERE/_ref" python -c "import whff; assert whff.BACKEND_NAME == 'compiled', whff.BACKEND_NAME; print('oracle/_ref: whff', whff.__version__, whff.BACKEND_NAME)"
