#!/bin/sh
# Copy the reference package's own test suite (read-only source at
# /root/reference/pkg/tests) to baseline/_ref_tests/ -- git-ignored, but not
# gpurun-ignored, so it travels to the GPU box with the snapshot, where
# tests/test_reference_suite.py runs it against this build through the
# `lpic` import name (lpic/__init__.py).  Nothing is committed from it.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg/tests
DST="$ROOT/baseline/_ref_tests"
[ -d "$SRC" ] || { echo "no reference tests at $SRC" >&2; exit 1; }
rm -rf "$DST"
mkdir -p "$DST"
cp "$SRC"/*.py "$DST"/
echo "copied $(ls "$DST" | wc -l) files to $DST"
