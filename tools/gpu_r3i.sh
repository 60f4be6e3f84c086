#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for r in 1 2 3; do
timeout 600 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_q$r.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_q$r.json'));print('run $r',j['value'],j['ms_per_step'],j['wall_s_timed_loop'],j['e2e']['value'],j['roofline']['kernel'],j['roofline']['frac'])"
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python -c "import json;j=json.load(open('gpurun_out/bench_default.json'));print(j['value'],j['ms_per_step'],j['e2e']['value'],j['roofline']['kernel'],j['roofline']['frac'],j['c4']['ms_per_iter'],j['c4']['spmm_gate']['frac'],j['c4']['spmm_gate'].get('dram_frac'))"
