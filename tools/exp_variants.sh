mkdir -p gpurun_out
run() { tag=$1; shift; timeout 300 env "$@" > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/exp_$tag.json'))
print('$tag', 'value %.4g k_sim %.3f ms disp %d events %d' % (d['value'], d['kernel_ms']['k_sim_mean'], d['config']['dispatches_per_step_per_gpu'], d['config']['events_per_step']))" 2>&1 | tail -1; }
run base python bench.py --no-cpu-baseline --steps 5 --e2e-steps 1
run nosync GFQ_LIB=paper_2507_08954_b200/var_nosync.so python bench.py --no-cpu-baseline --steps 5 --e2e-steps 1
GFQ_LIB=paper_2507_08954_b200/var_nosync.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "golden_family or fast_build" 2>&1 | tail -2
