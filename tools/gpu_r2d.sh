#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-c4 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench=$?; tail -2 gpurun_out/bench_c5.err
python - <<'PY'
import json
j = json.load(open("gpurun_out/bench_c5.json")); print(j["value"], j["ms_per_step"], j.get("e2e", {}).get("value"), j.get("gpu_launches"), j["dp_checks"].get("oracle_grad_row_err_max"))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c4 > /dev/null 2>&1; echo ncu=$?
