#!/bin/bash
# ncu --set full of the C4 D-ReLU (cell) kernel; raw + source CSV exported on the box.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:drelu -c 1 \
  -o /tmp/full_drelu python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_drelu.log 2>&1
echo rc=$?
ncu -i /tmp/full_drelu.ncu-rep --page raw --csv > gpurun_out/full_drelu_raw.csv 2>/dev/null
ncu -i /tmp/full_drelu.ncu-rep --page source --csv --print-source sass > gpurun_out/full_drelu_sass.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/full_drelu_raw.csv | cut -c1-220 | head -60
