#!/bin/bash
mkdir -p gpurun_out
for w in 8 4 2 8 4 2; do
DR_SPMM_WPC=$w timeout 300 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_w$w.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_w$w.json'));k=j['kernels'];print('wpc=$w',j['value'],j['ms_per_step'],{t:k[t]['mean_ms'] for t in k if 'spmm' in t})"
done
