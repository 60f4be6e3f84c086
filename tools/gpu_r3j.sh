#!/bin/bash
mkdir -p gpurun_out
for q in 1 2 3; do
timeout 300 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_l$q.json 2> gpurun_out/bench_l.err
python -c "import json;j=json.load(open('gpurun_out/bench_l$q.json'));print('run $q',j['value'],j['ms_per_step'],j['step_ms_rank0'],j['clocks'])"
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python -c "import json;j=json.load(open('gpurun_out/bench_default.json'));print(j['value'],j['ms_per_step'],j['step_ms_rank0'],j['e2e']['value'],j['roofline']['kernel'],j['roofline']['frac'],j['c4']['ms_per_iter'],j['c4']['spmm_gate']['frac'],j['c4']['spmm_gate'].get('dram_frac'))"
