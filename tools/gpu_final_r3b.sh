#!/bin/bash
# final check of session 3: smoke, full GPU tests, default bench, sanitizers on the new paths
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python -c "import json;j=json.load(open('gpurun_out/bench_default.json'));print(j['value'],j['ms_per_step'],j['step_ms_rank0'],j['e2e']['value'],j['roofline']['kernel'],j['roofline']['frac'],j['c4']['ms_per_iter'],j['c4']['spmm_gate']['frac'],j['c4']['spmm_gate'].get('dram_frac'))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c4 > /dev/null 2>&1; echo l5=$?
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1; echo $tool=$?; tail -3 gpurun_out/sanitize_$tool.log
done
DR_TC2_EWG=2 timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_memcheck_ewg2.log 2>&1; echo memcheck_ewg2=$?; tail -2 gpurun_out/sanitize_memcheck_ewg2.log
