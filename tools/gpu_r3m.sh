#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "heteroconv or train or chain or fullsize" 2>&1 | tail -3
for q in 1 0 1 0; do
DR_DW_DUAL=$q timeout 300 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_d$q.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_d$q.json'));k=j['kernels'];print('dual=$q',j['value'],j['ms_per_step'],j['dp_checks']['oracle_grad_row_err_max'],{t:k[t]['mean_ms'] for t in k if 'dw' in t})"
done
