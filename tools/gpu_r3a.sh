#!/bin/bash
# re-entry check: smoke, GPU tests, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python -c "import json;j=json.load(open('gpurun_out/bench_default.json'));print(j['value'],j['ms_per_step'],j['e2e']['value'],j['roofline']['kernel'],j['roofline']['frac'],j['c4']['ms_per_iter'],j['c4']['spmm_gate']['frac'],j['c4']['spmm_gate'].get('dram_frac'))"
