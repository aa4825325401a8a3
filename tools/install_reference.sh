#!/bin/bash
# Install the UNMODIFIED reference under baseline/_ref (git-ignored, shipped to the
# GPU box by gpurun) and copy its test files beside it (tests/test_gpu_dropin.py,
# bench.py --impl reference, tools/cpu_baselines.py).  DESIGN.md section 9.
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC; keeping the existing baseline/_ref" >&2; exit 0; }
[ -d "$ROOT/baseline/_ref/fieldfit" ] && [ -d "$ROOT/baseline/_ref/tests_ref" ] && exit 0
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"            # the build writes into its source tree; /root/reference is read-only
mkdir -p "$ROOT/baseline"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/tests_ref"
cp "$SRC"/tests/*.py "$SRC"/pytest.ini "$ROOT/baseline/_ref/tests_ref/"
rm -rf "$TMP"
