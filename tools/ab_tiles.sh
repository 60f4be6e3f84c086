#!/bin/bash
# tiled (tensor-core) vs SIMT SpMM on C2 and C4, plus tspmm role timers; spmm GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tspmm.py tests/test_gpu_parity.py -x -q -k "tspmm or spmm or heteroconv or train" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 300 python profiles/spmm_ab.py C2 default DR_TSPMM=0 > gpurun_out/ab_tiles_c2.txt 2>&1
DR_TS_DEBUG=1 timeout 300 python profiles/spmm_ab.py C2 default > gpurun_out/dbg_c2.txt 2>&1
timeout 600 python profiles/spmm_ab.py C4 default DR_TSPMM=0 > gpurun_out/ab_tiles_c4.txt 2>&1
DR_TS_DEBUG=1 timeout 600 python profiles/spmm_ab.py C4 default > gpurun_out/dbg_c4.txt 2>&1
for f in gpurun_out/dbg_c2.txt gpurun_out/dbg_c4.txt; do grep -h "tspmm fwd" $f | head -1; grep -h "tspmm bwd" $f | head -1; done
python - <<'PY'
import json
for f in ['gpurun_out/ab_tiles_c2.txt','gpurun_out/ab_tiles_c4.txt']:
    for line in open(f):
        if line.startswith('default') or line.startswith('DR_TSPMM'):
            name, js = line.split(' ',1); j=json.loads(js); sk=j['seq_kernels_ms']
            print(f[-6:-4], name, 'layer', j['layer.fwd_bwd'], {k:v for k,v in sk.items() if 'spmm' in k}, 'sum', round(sum(sk.values()),3))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python profiles/summarize.py gpurun_out/launches_c2.csv 2 | head -20
