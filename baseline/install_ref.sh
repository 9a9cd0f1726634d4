#!/bin/bash
# Install the UNMODIFIED reference package under git-ignored baseline/_ref
# (travels to the GPU box with the gpurun snapshot).  /root/reference is
# read-only, so the build runs from a copy under /tmp.
set -eu
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg}
[ -f "$HERE/_ref/sortlab/sort_core.py" ] && exit 0
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 0; }
TMP=$(mktemp -d /tmp/ref_pkg.XXXXXX)
cp -r "$SRC"/. "$TMP"/
python -m pip install -q --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP"
rm -rf "$TMP"
