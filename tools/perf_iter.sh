#!/bin/bash
# One gpurun call per kernel change: smoke, C3 bench (no CPU leg), then the GPU parity suite.
#   gpurun --timeout 1500 -- bash tools/perf_iter.sh <tag> [bench args...]
tag=${1:-it}; shift
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.log
timeout 180 python bench.py --no-cpu-baseline "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${tag}_bench.json'))
print('value %.4g e2e %.4g k_sim %.3f ms step %.3f ms launches %d clocks %s' % (d['value'], d['e2e']['value'], d['kernel_ms']['k_sim_mean'], d['ms_per_step'], d['gpu_launches'], d['clocks']))" 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${tag}_pytest.log
