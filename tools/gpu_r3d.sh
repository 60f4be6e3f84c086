#!/bin/bash
# A/B: rolled-chunk (stream) vs unrolled thread-per-row network; C5 bench both ways
mkdir -p gpurun_out
python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -2
timeout 300 python tools/drelu_ab.py > gpurun_out/drelu_ab3.json 2>&1; echo ab=$?; cat gpurun_out/drelu_ab3.json
for s in 0 1 0 1; do
DR_TPR_STREAM=$s timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-c4 > gpurun_out/bench_s$s.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_s$s.json'));k=j['kernels'];print('stream=$s',j['value'],j['ms_per_step'],{t:k[t]['mean_ms'] for t in k if 'proj' in t})"
done
DR_NO_GRAPH=1 DR_TC2_DEBUG=1 timeout 300 python tools/c5_step.py 1 2>&1 | grep "tc2_rows" | tail -5 | cut -c1-300
