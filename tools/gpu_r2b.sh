#!/bin/bash
# round 2: fused next-layer D-ReLU (a5) + dead last-layer Y_net: new tests, full GPU suite, C5 bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q > gpurun_out/pytest_chain.log 2>&1; echo chain=$?; tail -15 gpurun_out/pytest_chain.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-c4 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench=$?; tail -3 gpurun_out/bench_c5.err
DR_CHAIN=0 DR_SKIP_DEAD_NET=0 timeout 600 python bench.py --no-c4 --no-cpu-baseline > gpurun_out/bench_c5_nochain.json 2> gpurun_out/bench_c5_nochain.err; echo bench0=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench_c5.json", "gpurun_out/bench_c5_nochain.json"):
    try:
        j = json.load(open(f)); print(f, j["value"], j["ms_per_step"], j.get("e2e", {}).get("value"), j.get("gpu_launches"))
    except Exception as e: print(f, "ERR", e)
PY
