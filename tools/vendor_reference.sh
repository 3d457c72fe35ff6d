#!/bin/bash
# Install the UNMODIFIED reference (moesim) under baseline/_ref (git-ignored, but it travels to the
# GPU box with the gpurun snapshot), with its run configs, so its engine, scheduler and chunk bench
# can drive the GPU layer there (paper_2510_08055_b200/refdrive.py). The build needs a writable
# tree, so it installs from a copy under /tmp; /root/reference stays read-only.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { cat "$TMP/pip.log"; exit 1; }
cp -r "$SRC/configs" "$ROOT/baseline/_ref/configs"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import moesim, moesim.engine; print('moesim', moesim.__file__)"
