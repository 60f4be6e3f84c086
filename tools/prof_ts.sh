#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
B="python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tspmm_kernel -s 1 -c 1 -o /tmp/tsb $B > gpurun_out/ncu_tsb.log 2>&1
ncu -i /tmp/tsb.ncu-rep --page source --csv --print-source sass > gpurun_out/src_tsb.csv 2>/dev/null
ncu -i /tmp/tsb.ncu-rep --page raw --csv > gpurun_out/raw_tsb.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/raw_tsb.csv | tail -1 | cut -c1-200
