#!/bin/bash
# Installs the UNMODIFIED reference package (lb2d: pure Python, numba backend) into
# baseline/_ref/ (git-ignored, travels to the GPU box with the snapshot) so that
# bench.py can time it there as `cpu_baseline_ref2d`.  The reference tree is
# read-only and setuptools writes build files next to pyproject.toml, so the
# install runs from a scratch copy; dependencies (numpy, numba) are already in
# the image, hence --no-deps.  Nothing from the reference enters the repository.
set -eu
HERE="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference tree at $SRC: nothing to install"; exit 0; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$HERE/baseline/_ref" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { tail -20 "$TMP/pip.log"; exit 1; }
rm -rf "$TMP"
echo "installed lb2d into $HERE/baseline/_ref"
