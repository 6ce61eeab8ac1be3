mkdir -p gpurun_out
run() { tag=$1; shift; timeout 200 env "$@" > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/exp_$tag.json'))
print('$tag', 'value %.4g k_sim %.3f ms k_reduce %.3f' % (d['value'], d['kernel_ms']['k_sim_mean'], d['kernel_ms']['k_reduce_mean']))" 2>&1 | tail -1; }
run c3 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 1
run c4 python bench.py --no-cpu-baseline --steps 3 --e2e-steps 1 --workload c4
run c4none GFQ_LIB=paper_2507_08954_b200/var_none.so python bench.py --no-cpu-baseline --steps 3 --e2e-steps 1 --workload c4
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
