#!/bin/bash
# Stage the reference package (sources + its tests) into the git-ignored
# baseline/_ref so a gpurun snapshot carries it to the GPU box, where
# tools/run_reference_suite.sh runs the reference's own tests with the
# B200 operator swapped in.  Run in the build container (it reads
# /root/reference); nothing staged here is committed.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf "$ROOT/baseline/_ref/pkg"
mkdir -p "$ROOT/baseline/_ref/pkg"
cp -r /root/reference/pkg/src /root/reference/pkg/tests "$ROOT/baseline/_ref/pkg/"
find "$ROOT/baseline/_ref" -name __pycache__ -prune -exec rm -rf {} +
echo "staged $(find "$ROOT/baseline/_ref/pkg" -name '*.py' | wc -l) files into baseline/_ref/pkg"
