#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "heteroconv or dense or train" > gpurun_out/pytest_dw.log 2>&1; echo dw=$?; tail -3 gpurun_out/pytest_dw.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-c4 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench=$?; tail -2 gpurun_out/bench_c5.err
python - <<'PY'
import json
j = json.load(open("gpurun_out/bench_c5.json")); print(j["value"], j["ms_per_step"], j.get("gpu_launches"), j["dp_checks"].get("oracle_grad_row_err_max"))
print({k: v["mean_ms"] for k, v in j["kernels"].items() if "dw" in k})
PY
