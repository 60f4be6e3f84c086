#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python - <<'PY'
import json
for f in ['gpurun_out/bench_c2.json','gpurun_out/bench_c4.json']:
    j=json.load(open(f))
    print(f, j['value'], j['unit'], j['ms_per_step'], 'launches/step', j['gpu_launches']/j['steps'], 'e2e', (j['e2e'] or {}).get('value'))
    print(' roofline', j['roofline'])
    ks=j['kernels']; tot=sum(v['total_ms'] for v in ks.values())
    for t,v in sorted(ks.items(), key=lambda x:-x[1]['total_ms'])[:8]: print('  %-22s %8.4f ms  %5.1f%%  gbs=%s'%(t,v['mean_ms'],100*v['total_ms']/tot,v['gbs']))
    print(' sum kernels per step', round(tot/j['steps'],4))
PY
