#!/bin/bash
# Install the UNMODIFIED reference (pab-engine, pure Python) into oracle/_ref/ so the
# bench's reference arm (bench.py --impl reference) can time the reference's own code
# on the GPU box, where /root/reference does not exist.  oracle/_ref/ is git-ignored
# (never committed) but travels to the box with the gpurun snapshot.
# Test/bench infrastructure only: the product path never imports it.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${PAB_REFERENCE_PKG:-/root/reference/pkg}
[ -d "$SRC/src/pab_engine" ] || { echo "reference not found at $SRC (nothing to do)"; exit 0; }
rm -rf "$HERE/_ref"
mkdir -p "$HERE/_ref"
# the source tree is read-only: build from a scratch copy
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
if ! python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg" \
      > "$TMP/pip.log" 2>&1; then
  # no wheel tooling: the package is pure Python, a verbatim copy of src/ is the install
  cp -r "$TMP/pkg/src/pab_engine" "$HERE/_ref/pab_engine"
fi
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import pab_engine, os; print('reference installed:', os.path.dirname(pab_engine.__file__))"
