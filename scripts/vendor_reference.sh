#!/usr/bin/env bash
# Install the UNMODIFIED reference package (traceobf 0.1.0, /root/reference/pkg)
# into baseline/_ref — the one offline install the task allows. Built from a
# copy under /tmp (the build writes into its source tree; /root/reference is
# read-only); --no-deps: its only dependency, numpy, is already in the image
# and not in the wheelhouse. baseline/_ref is git-ignored but travels to the
# GPU box with every gpurun snapshot (used by bench.py --impl reference and the
# drop-in tests there, where /root/reference does not exist).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d /tmp/traceobf_src.XXXXXX)"
cp -r "$SRC"/. "$TMP"/
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP"
rm -rf "$TMP"
python - "$ROOT/baseline/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import traceobf
print("vendored traceobf", traceobf.__version__, "->", traceobf.__file__)
PY
