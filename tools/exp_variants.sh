mkdir -p gpurun_out
run() { tag=$1; shift; timeout 300 env "$@" > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/exp_$tag.json'))
print('$tag', 'value %.4g k_sim %.3f ms' % (d['value'], d['kernel_ms']['k_sim_mean']), {k:v for k,v in d['config'].items() if k in ('window_memo_hits','window_memo_misses','ticks')})" 2>&1 | tail -1; }
run base python bench.py --no-cpu-baseline --steps 10 --e2e-steps 1
run diag GFQ_LIB=paper_2507_08954_b200/var_diag.so python bench.py --no-cpu-baseline --steps 3 --e2e-steps 1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -1
