#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "chain or train or head or fullsize" 2>&1 | tail -2
for r in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_h.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_h.json'));k=j['kernels'];print(j['value'],j['ms_per_step'],j['dp_checks']['oracle_grad_row_err_max'],j['step0_loss'],{t:k[t]['mean_ms'] for t in k if 'proj' in t or 'head' in t})"
done
