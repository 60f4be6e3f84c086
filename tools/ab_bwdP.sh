#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -k "spmm_bwd or heteroconv" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for P in 1 2 4; do DR_BWD_P=$P timeout 300 python profiles/spmm_ab.py C4 default 2>&1 | grep -o '"spmm_bwd[^,]*,[^,]*,' | tr '\n' ' '; echo " P=$P C4"; done
for P in 1 2 4; do DR_BWD_P=$P timeout 300 python profiles/spmm_ab.py C2 default 2>&1 | grep -o '"spmm_bwd[^,]*,[^,]*,' | tr '\n' ' '; echo " P=$P C2"; done
