#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "chain or heteroconv or train or head or dense or split" 2>&1 | tail -3
DR_NO_GRAPH=1 DR_TC2_DEBUG=1 timeout 300 python tools/c5_step.py 1 2>&1 | grep "tc2_rows" | tail -10 | cut -c1-300
for e in 2 1 2 1; do
DR_TC2_EWG=$e timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-c4 > gpurun_out/bench_e$e.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_e$e.json'));k=j['kernels'];print('ewg=$e',j['value'],j['ms_per_step'],j['e2e']['ms_per_step'],{t:k[t]['mean_ms'] for t in k if 'tc_' in t})"
done
