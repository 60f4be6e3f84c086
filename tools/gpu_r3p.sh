#!/bin/bash
mkdir -p gpurun_out
DR_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:drelu_tcoop" -s 0 -c 1 -o /tmp/dr python tools/c5_step.py 1 > gpurun_out/ncu_dr.log 2>&1; echo ncu=$?
ncu -i /tmp/dr.ncu-rep --page raw --csv > gpurun_out/raw_dr.csv 2>/dev/null
ncu -i /tmp/dr.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/mix_dr.csv 2>/dev/null
ncu -i /tmp/dr.ncu-rep --page source --csv --print-source sass > gpurun_out/src_dr.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/raw_dr.csv | cut -c1-220
python profiles/line_hot.py gpurun_out/mix_dr.csv 25
