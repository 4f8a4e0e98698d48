#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (`segconv`, /root/reference/pkg) into baseline/_ref
# (git-ignored; it travels to the GPU box with the repo snapshot), plus a copy of the reference's
# own test suites under baseline/_ref/tests, for:
#   - bench.py --impl reference   (times the reference's own CPU engine, kind "reference")
#   - tests/test_gpu_reference_suite.py  (runs the reference's test_engines.py /
#     test_acceptance.py / test_segregation.py with its segregated engine routed to the B200
#     path through integration/segconv_gpu.py, INTEGRATION.md option B)
# The offline install the task allows (no index; dependencies are already in the image).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "reference package not found at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"   # the build writes egg-info next to the sources; the reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
mkdir -p "$ROOT/baseline/_ref/tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/tests/"
rm -rf "$TMP"
echo "installed segconv into $ROOT/baseline/_ref ($(ls "$ROOT/baseline/_ref/tests" | wc -l) test files)"
