#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "drelu or c4_full or c2_full" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
for C in C4 C2; do
timeout 600 python profiles/spmm_ab.py $C default > gpurun_out/ab_$C.txt 2>&1
python - $C <<'PY'
import json,sys
for line in open('gpurun_out/ab_%s.txt'%sys.argv[1]):
    if line.startswith('default'):
        name, js = line.split(' ',1); j=json.loads(js); sk=j['seq_kernels_ms']
        print(sys.argv[1], 'layer', j['layer.fwd_bwd'], {k:v for k,v in sk.items() if 'drelu' in k})
PY
done
