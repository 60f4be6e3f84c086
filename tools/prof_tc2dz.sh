#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1

timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_rows -s 4 -c 1 -o /tmp/dz python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dz.log 2>&1
ncu -i /tmp/dz.ncu-rep --page raw --csv > gpurun_out/dz_raw.csv 2>/dev/null
ncu -i /tmp/dz.ncu-rep --page source --csv --print-source sass > gpurun_out/dz_src.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/dz_raw.csv | cut -c1-250
