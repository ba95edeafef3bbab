#!/bin/bash
# Install the unmodified reference (simtdg, pure Python) into baseline/_ref for `bench.py --impl reference`
# and the cpu_baseline leg.  The reference tree is read-only, so pip builds from a copy under /tmp.
# baseline/_ref is git-ignored but not gpurun-ignored: it travels to the GPU box with the snapshot.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference tree at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import simtdg; print('simtdg', simtdg.__version__, 'installed')"
