#!/bin/bash
# inner loop: build, GPU tests, C4/C2 per-kernel times and tc2 role timers
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
DR_TC2_DEBUG=1 timeout 600 python profiles/spmm_ab.py C4 default > gpurun_out/dbg_tc2_c4.txt 2>&1
grep -h "tc2_rows\|tc2_reduce" gpurun_out/dbg_tc2_c4.txt | sort | uniq | awk '!seen[substr($0,1,60)]++' | head -12
for C in C4 C2; do
timeout 600 python profiles/spmm_ab.py $C default > gpurun_out/ab_$C.txt 2>&1
python - $C <<'PY'
import json,sys
for line in open('gpurun_out/ab_%s.txt'%sys.argv[1]):
    if line.startswith('default'):
        name, js = line.split(' ',1); j=json.loads(js); sk=j['seq_kernels_ms']
        print(sys.argv[1], 'layer', j['layer.fwd_bwd'], 'sum', round(sum(sk.values()),3), sk)
PY
done
