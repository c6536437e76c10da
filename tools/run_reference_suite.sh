#!/bin/bash
# On a GPU box: the reference's own tests (staged by stage_reference.sh)
# with paper_2302_05164_b200.ThermalOperator swapped in
# (tests/refswap/refswap_plugin.py).  Output: gpurun_out/refsuite.txt
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF="$ROOT/baseline/_ref/pkg"
if [ ! -d "$REF/tests" ]; then echo "reference not staged (tools/stage_reference.sh)"; exit 2; fi
mkdir -p "$ROOT/gpurun_out"
cd "$REF/tests"
PYTHONPATH="$REF/src:$ROOT:$ROOT/tests/refswap" timeout ${REFSUITE_TIMEOUT:-2400} \
  python -m pytest -p refswap_plugin -p no:cacheprovider -q -rA "$@" \
  > "$ROOT/gpurun_out/refsuite.txt" 2>&1
rc=$?
echo "refsuite rc=$rc" >> "$ROOT/gpurun_out/refsuite.txt"
tail -40 "$ROOT/gpurun_out/refsuite.txt"
