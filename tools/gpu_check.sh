#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (N=1), launch list and one ncu --set full of k_sim.
#   gpurun --timeout 2400 -- bash tools/gpu_check.sh <tag> [bench args...]
# SKIP_TESTS=1 skips pytest + smoke.
tag=${1:-run}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_gpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
fi
timeout 900 python bench.py "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 "$@" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sim -s 1 -c 1 \
    -o gpurun_out/${tag}_k_sim -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/${tag}_ncu.log 2>&1
tail -3 gpurun_out/${tag}_pytest.log 2>/dev/null; tail -2 gpurun_out/${tag}_smoke.log 2>/dev/null; cat gpurun_out/${tag}_bench.json
