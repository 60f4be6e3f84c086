#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "chain or heteroconv or train or head or dense or split" 2>&1 | tail -2
for e in 0 1; do
DR_TC2_EWG=$e timeout 300 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_e$e.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_e$e.json'));k=j['kernels'];print('ewg=$e',j['value'],j['ms_per_step'],{t:k[t]['mean_ms'] for t in k if 'tc_' in t})"
DR_TC2_EWG=$e timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4e$e.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_c4e$e.json'));k=j['kernels'];print('C4 ewg=$e',j['ms_per_step'],{t:k[t]['mean_ms'] for t in k if 'tc_' in t})"
done
