#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tspmm.py tests/test_gpu_parity.py -x -q -k "tspmm or spmm or heteroconv or train" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
for C in C2 C4; do
DR_TS_DEBUG=1 timeout 600 python profiles/spmm_ab.py $C default > gpurun_out/dbg_$C.txt 2>&1
grep "tspmm" gpurun_out/dbg_$C.txt | sort | uniq -c | sort -rn | awk '{$1="";print}' | sort -u | grep -v "kcycles/CTA: total" | head -4
grep "tspmm" gpurun_out/dbg_$C.txt | grep "kcycles/CTA: total" | sort -u | tail -2
timeout 600 python profiles/spmm_ab.py $C default > gpurun_out/ab_$C.txt 2>&1
python - $C <<'PY'
import json,sys
for line in open('gpurun_out/ab_%s.txt'%sys.argv[1]):
    if line.startswith('default') or line.startswith('DR_'):
        name, js = line.split(' ',1); j=json.loads(js); sk=j['seq_kernels_ms']
        print(sys.argv[1], name, 'layer', j['layer.fwd_bwd'], {k:v for k,v in sk.items() if 'spmm' in k}, 'sum', round(sum(sk.values()),3))
PY
done
