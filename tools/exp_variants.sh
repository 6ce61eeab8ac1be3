mkdir -p gpurun_out
run() { tag=$1; shift; timeout 300 env "$@" > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/exp_$tag.json'))
print('$tag', 'value %.4g k_sim %.3f ms' % (d['value'], d['kernel_ms']['k_sim_mean']))" 2>&1 | tail -1; }
run base python bench.py --no-cpu-baseline --steps 10 --e2e-steps 1
run aeo GFQ_LIB=paper_2507_08954_b200/var_aeo.so python bench.py --no-cpu-baseline --steps 10 --e2e-steps 1
run o2 GFQ_LIB=paper_2507_08954_b200/var_o2.so python bench.py --no-cpu-baseline --steps 10 --e2e-steps 1
run base2 python bench.py --no-cpu-baseline --steps 10 --e2e-steps 1
