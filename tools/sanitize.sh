#!/bin/bash
# compute-sanitizer over every build on a small random batch (one gpurun call):
#   gpurun --timeout 2400 -- bash tools/sanitize.sh
mkdir -p gpurun_out
run() { tool=$1; shift; timeout 900 compute-sanitizer --tool $tool "$@" python tools/sanitize_batch.py 10 \
        > gpurun_out/sanitize_$tool.txt 2>&1; echo "$tool rc=$?"; grep -E "SUMMARY" gpurun_out/sanitize_$tool.txt; }
run memcheck --print-limit 20
run initcheck --print-limit 20
run synccheck --print-limit 20
run racecheck --racecheck-detect-level error --print-limit 20
