mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
GFQ_LIB=paper_2507_08954_b200/var_strict.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
timeout 300 python bench.py --no-cpu-baseline --steps 10 --e2e-steps 3 > gpurun_out/exp_b.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/exp_b.json'))
print('value %.4g e2e %.4g k_sim %.3f ms' % (d['value'], d['e2e']['value'], d['kernel_ms']['k_sim_mean']))"
