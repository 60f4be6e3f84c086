#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q > gpurun_out/pytest_chain.log 2>&1; echo chain=$?; tail -5 gpurun_out/pytest_chain.log
python tools/chain_prof.py 20 > gpurun_out/chainprof.txt 2>&1; cat gpurun_out/chainprof.txt | tail -2
DR_TC2_DEBUG=1 python tools/chain_prof.py 1 2>&1 | grep "tc2_rows" | sort | uniq | cut -c1-300
timeout 600 python bench.py --no-c4 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench=$?; tail -2 gpurun_out/bench_c5.err
DR_CHAIN=0 timeout 600 python bench.py --no-c4 --no-cpu-baseline > gpurun_out/bench_c5_nochain.json 2> gpurun_out/bench_c5_nochain.err; echo bench0=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench_c5.json", "gpurun_out/bench_c5_nochain.json"):
    try:
        j = json.load(open(f)); print(f, j["value"], j["ms_per_step"], j.get("e2e", {}).get("value"), j.get("gpu_launches"), j["dp_checks"].get("oracle_grad_row_err_max"))
        print({k: v["mean_ms"] for k, v in j["kernels"].items() if "proj" in k or "drelu" in k})
    except Exception as e: print(f, "ERR", e)
PY
