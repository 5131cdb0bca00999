timeout 300 python tests/gpu_debug_bwd.py 2>&1 | tail -8
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'clk', d['clocks'])
for k,v in d['kernels'].items(): print(k, round(v['ms'],2), v['alg_tflops'] and round(v['alg_tflops'],1), v['executed_tflops'] and round(v['executed_tflops'],1))"
