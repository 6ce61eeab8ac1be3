#!/usr/bin/env bash
# Install the UNMODIFIED reference (gpufairq, pure Python) into baseline/_ref
# -- git-ignored, not gpurun-ignored, so it travels to the GPU box -- with its
# own test suite and configs beside it (baseline/_ref/refpkg/{tests,configs}).
# Used only as a checker / baseline: the reference-suite shim tests
# (tests/test_gpu_reference_suite.py), the drop-in comparison tests and the
# bench's Python-reference CPU sample.  Run in the build container (where
# /root/reference exists); the product never imports it.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${REF:-/root/reference/pkg}"
DEST="$ROOT/baseline/_ref"
rm -rf "$DEST" /tmp/gfq_refbuild
mkdir -p "$DEST"
cp -r "$REF" /tmp/gfq_refbuild          # the build writes egg-info: never into /root/reference
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$DEST" /tmp/gfq_refbuild
mkdir -p "$DEST/refpkg"
cp -r "$REF/tests" "$REF/configs" "$DEST/refpkg/"
rm -rf /tmp/gfq_refbuild
python - "$DEST" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import gpufairq
print("installed", gpufairq.__file__, gpufairq.__version__)
PY
