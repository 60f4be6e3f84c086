#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
cat > /tmp/t.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch, numpy as np, paper_2508_16769_b200 as dr
from gen import make_config
d = make_config("C2", scale=0.1)
g = dr.Graph.from_design(d)
x = torch.randn(d.n_cell, 64, device="cuda")
v, i = dr.drelu_topk(x, 8)
z = dr.spmm_fwd(g, "near", v, i, 64)
torch.cuda.synchronize()
PY
DR_NVTX=1 ncu --nvtx --print-nvtx-rename kernel --metrics gpu__time_duration.sum --csv python /tmp/t.py 2>&1 | grep -v "^==PROF" | tail -5
timeout 900 python -m pytest tests -m gpu -x -q -k "drelu or heteroconv or train" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 600 python profiles/spmm_ab.py C4 default > gpurun_out/ab_C4.txt 2>&1
python - C4 <<'PY'
import json,sys
for line in open('gpurun_out/ab_%s.txt'%sys.argv[1]):
    if line.startswith('default'):
        name, js = line.split(' ',1); j=json.loads(js); sk=j['seq_kernels_ms']
        print(sys.argv[1], name, 'layer', j['layer.fwd_bwd'], {k:v for k,v in sk.items() if 'drelu' in k})
PY
