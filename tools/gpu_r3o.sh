#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_push.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_push.log | grep -v "^\.\.\." | tail -12
for q in 1 0; do
DR_DZ_PUSH=$q timeout 300 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_p$q.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_p$q.json'));k=j['kernels'];print('push=$q',j['value'],j['ms_per_step'],j['dp_checks']['oracle_grad_row_err_max'],{t:k[t]['mean_ms'] for t in k if 'pinned' in t or '.net' in t})"
DR_DZ_PUSH=$q timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4p$q.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_c4p$q.json'));k=j['kernels'];print('C4 push=$q',j['ms_per_step'],{t:(k[t]['mean_ms'],k[t]['alg_gbs']) for t in k if 'pinned' in t or '.net' in t})"
done
