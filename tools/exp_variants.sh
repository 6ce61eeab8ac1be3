mkdir -p gpurun_out
run() { tag=$1; shift; timeout 300 env "$@" > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/exp_$tag.json'))
print('$tag', 'value %.4g e2e %.4g k_sim %.3f ms k_reduce %.3f' % (d['value'], d['e2e']['value'], d['kernel_ms']['k_sim_mean'], d['kernel_ms']['k_reduce_mean']))" 2>&1 | tail -1; }
run c5 python bench.py --no-cpu-baseline --steps 3 --workload c5
run c2 python bench.py --no-cpu-baseline --steps 5 --workload c2
run c4 python bench.py --no-cpu-baseline --steps 3 --workload c4
