#!/usr/bin/env bash
# Build the UNMODIFIED reference package (voxpipe 0.1.0, Python + Cython hash
# core) from /root/reference into oracle/_ref/ — test/baseline infrastructure
# only. /root/reference is read-only, so the build happens on a /tmp copy;
# outputs land only in oracle/_ref/ (git-ignored, NOT gpurun-ignored, so the
# built reference travels to the GPU box and `bench.py --impl reference` can
# time the reference's own CPU path there). No reference source is committed.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${VOXPIPE_REF_SRC:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference not present at $SRC; keeping existing oracle/_ref" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/vxref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$OUT" "$TMP/pkg"
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
from voxpipe import kernels
assert kernels.backend_name() == "compiled", kernels.backend_name()
print("oracle/_ref: voxpipe built, backend", kernels.backend_name())
PY
