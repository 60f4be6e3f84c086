mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "
import json;j=json.load(open('gpurun_out/bench_c2.json'));print('C2',j['value'],j['ms_per_step'],j['e2e']['value'])
ks=j['kernels']
print({k:v['mean_ms'] for k,v in ks.items() if k.startswith('tc_dw')})"
done
