#!/usr/bin/env bash
# Build the UNMODIFIED reference CPU package (batchbleu + batchbleu_ext) into
# oracle/_ref/ so it can act as the checker and the CPU baseline.
#
# Test/bench infrastructure only: nothing in paper_2510_05485_b200/ imports it.
# The reference tree (/root/reference) is read-only and its build writes into
# the source tree, so it is built from a scratch copy under /tmp and only the
# installed result lands in oracle/_ref/ (git-ignored, but it travels to the
# GPU box with the gpurun snapshot).  No reference source is committed.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REFERENCE_ROOT:-/root/reference}"
OUT="$HERE/_ref"
if [ ! -d "$REF/pkg" ]; then
  echo "reference tree $REF/pkg not present; keeping existing $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/tbref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF/pkg" "$TMP/pkg"
rm -rf "$OUT"
mkdir -p "$OUT"
PIP="python -m pip install --no-index --no-build-isolation --no-deps --quiet --target $OUT"
$PIP "$TMP/pkg"
# the bindings import batchbleu at build time only through cythonize (no import)
$PIP "$TMP/pkg/bindings"
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import batchbleu, batchbleu_ext
assert "compiled" in batchbleu.available_backends(), batchbleu.available_backends()
print("reference built:", batchbleu.__file__, batchbleu.available_backends())
PY
