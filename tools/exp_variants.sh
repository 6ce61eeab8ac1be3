mkdir -p gpurun_out
run() { tag=$1; shift; timeout 300 env "$@" > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/exp_$tag.json'))
print('$tag', 'value %.4g e2e %.4g k_sim %.3f ms k_reduce %.3f' % (d['value'], d['e2e']['value'], d['kernel_ms']['k_sim_mean'], d['kernel_ms']['k_reduce_mean']))" 2>&1 | tail -1; }
run c3 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 1
run c3b python bench.py --no-cpu-baseline --steps 5 --e2e-steps 1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_sim -s 1 -c 1 -o gpurun_out/exp_k_sim -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
