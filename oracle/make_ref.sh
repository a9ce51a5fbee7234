#!/usr/bin/env bash
# Stage the reference package (pure Python, /root/reference/pkg) into oracle/_ref so the GPU box
# -- where /root/reference does not exist -- can run it as the checker (tests/test_gpu_reference_suite.py)
# and as the CPU reference arm (bench.py --impl reference).  oracle/_ref is git-ignored (never
# committed) but travels with the gpurun snapshot.  Sources are copied unmodified; MANIFEST
# records their sha256.  Run from the build container: bash oracle/make_ref.sh
set -euo pipefail
SRC=${REF_ROOT:-/root/reference}/pkg
DST=$(cd "$(dirname "$0")" && pwd)/_ref
[ -d "$SRC/src/mixserve" ] || { echo "make_ref: no reference at $SRC" >&2; exit 1; }
rm -rf "$DST"
mkdir -p "$DST/src" "$DST/tests"
cp -r "$SRC/src/mixserve" "$DST/src/"
cp "$SRC"/tests/*.py "$DST/tests/"
find "$DST" -name __pycache__ -prune -exec rm -rf {} +
( cd "$DST" && find src tests -type f -name '*.py' | sort | xargs sha256sum ) > "$DST/MANIFEST"
echo "make_ref: staged $(wc -l < "$DST/MANIFEST") files from $SRC into $DST"
