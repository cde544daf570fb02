#!/usr/bin/env bash
# Install the UNMODIFIED reference package (latsum 0.1.0, /root/reference/pkg) into baseline/_ref
# for bench.py --impl reference.  Offline: no index, wheels only from /opt/wheelhouse; --no-deps
# because the reference's numba/mpmath floors are never imported by its code and
# numpy/scipy are already in the image.  The build writes an egg-info next to the sources, so it
# runs on a copy (/root/reference is read-only).  baseline/_ref is git-ignored but travels to the
# GPU box with the gpurun snapshot.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "reference sources not found at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import latsum; print('reference installed:', latsum.__file__)"
