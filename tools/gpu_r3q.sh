#!/bin/bash
mkdir -p gpurun_out
for q in 1 0 1 0; do
DR_SEQ=$q timeout 300 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_sq$q.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_sq$q.json'));print('seq=$q',j['value'],j['ms_per_step'],j['step_ms_rank0'])"
done
