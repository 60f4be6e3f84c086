#!/bin/bash
mkdir -p gpurun_out
for w in -1 1 2 4 -1 2; do
DR_TS_TILE_W=$w DR_TS_TILE_W_BWD=$w timeout 300 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_tw$w.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_tw$w.json'));k=j['kernels'];print('tile_w=$w',j['value'],j['ms_per_step'],{t:k[t]['mean_ms'] for t in k if 'near' in t and 'spmm' in t or 'cell' in t and 'spmm_bwd' in t})"
done
