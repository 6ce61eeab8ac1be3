#!/bin/bash
# Measurement of the batched experiment CLI: the same
# `sweep` / `compare` commands through this repo's CLI (one engine batch per
# command) and through the UNMODIFIED reference CLI (baseline/_ref, serial
# Python simulations), wall time each, and the output trees compared byte for
# byte (summary.json may differ in var_latency_s's last place, see INTEGRATION).
#   bash tools/cli_bench.sh [out.json]
set -u
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/cli_bench.json}
CFG=tests/golden/cli/default.cfg
TMP=$(mktemp -d)
T16=$(seq -s, 0 15)
T64=$(seq -s, 0 63)
declare -A CMDS=(
  [sweep_T16]="sweep --config $CFG --param T --values $T16"
  [sweep_T64_medium]="sweep --config tests/golden/cli/medium.cfg --param T --values $T64"
  [compare5]="compare --config $CFG --policies mqfq,fcfs,batch,sjf,fcfs_naive"
)
python -c "import paper_2507_08954_b200.engine" >/dev/null 2>&1   # warm the import / JIT
echo "{" > "$OUT"
first=1
for name in "${!CMDS[@]}"; do
  args=${CMDS[$name]}
  t0=$(date +%s.%N)
  python -m paper_2507_08954_b200.cli $args --out "$TMP/gpu_$name" > /dev/null 2>&1
  t1=$(date +%s.%N)
  PYTHONPATH=baseline/_ref python -m gpufairq.cli $args --out "$TMP/ref_$name" > /dev/null 2>&1
  t2=$(date +%s.%N)
  ndiff=$(diff -rq "$TMP/gpu_$name" "$TMP/ref_$name" | grep -v summary.json | wc -l)
  [ $first = 1 ] || echo "," >> "$OUT"; first=0
  python - "$name" "$t0" "$t1" "$t2" "$ndiff" "$args" >> "$OUT" <<'PY'
import json, sys
name, t0, t1, t2, nd, args = sys.argv[1], *map(float, sys.argv[2:5]), int(sys.argv[5]), sys.argv[6]
print(json.dumps(name) + ": " + json.dumps({"command": args, "gpu_cli_s": t1 - t0,
      "reference_cli_s": t2 - t1, "speedup": (t2 - t1) / (t1 - t0),
      "differing_files_except_summary_json": nd}), end="")
PY
done
echo "}" >> "$OUT"
# fixed costs of one CLI process here: interpreter + imports, and the CUDA context
python - >> "${OUT%.json}_startup.txt" <<'PY'
import time
t0 = time.perf_counter()
import paper_2507_08954_b200.cli  # noqa: F401
t1 = time.perf_counter()
from paper_2507_08954_b200.engine import Engine
Engine(0)
t2 = time.perf_counter()
print(f"import {t1 - t0:.3f} s, engine (CUDA context) {t2 - t1:.3f} s")
PY
cat "$OUT"
rm -rf "$TMP"
