#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (mwfloat, /root/reference/pkg)
# into baseline/_ref (git-ignored, NOT gpurun-ignored: it travels to the GPU
# box with the snapshot).  Run in the build container, where
# /root/reference exists; the GPU box only uses the installed copy.
#
#   baseline/_ref/mwfloat/      the reference package (+ its _fmaext C ufunc)
#   baseline/_ref/ref_tests/    the reference's own test tree, so that
#                               tests/test_reference_binding.py can run it
#                               against libmwgpu.so through the ctypes stub
#                               of INTEGRATION.md on the B200
#
# The build writes into the source tree, so it runs from a copy under /tmp
# (/root/reference is read-only).  Dependency resolution is skipped
# (--no-deps): numpy is already in the image.
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
DST="$REPO/baseline/_ref"
if [ ! -d "$SRC" ]; then
  echo "install_reference: $SRC not present (GPU box?) -- using the existing $DST" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/mwfloat_ref_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$DST"
mkdir -p "$DST"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$DST" "$TMP/pkg" >"$TMP/pip.log" 2>&1 || { cat "$TMP/pip.log" >&2; exit 1; }
cp -r "$SRC/tests" "$DST/ref_tests"
PYTHONPATH="$DST" python -c "import mwfloat, mwfloat._fmaext as f; print('mwfloat', mwfloat.__file__, f.fma(2.0**30 + 1, 2.0**30 + 1, -(2.0**60 + 2**31)))"
