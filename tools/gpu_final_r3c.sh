#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python -c "import json;j=json.load(open('gpurun_out/bench_default.json'));print(j['value'],j['ms_per_step'],j['step_ms_rank0'],j['e2e']['value'],j['roofline']['kernel'],j['roofline']['frac'],j['c4']['ms_per_iter'],j['c4']['spmm_gate']['frac'],j['c4']['spmm_gate'].get('dram_frac'),j['gpu_launches'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref=$?; head -c 300 gpurun_out/bench_reference.json
