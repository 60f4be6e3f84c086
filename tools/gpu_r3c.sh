#!/bin/bash
# C5: source-level stall profile of the fused-D-ReLU projection (L0 cell, tc2_rows_kernel<8>)
mkdir -p gpurun_out
DR_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc2_rows_kernel<\(int\)8>" -s 1 -c 1 -o /tmp/p8 python tools/c5_step.py 1 > gpurun_out/ncu_p8.log 2>&1; echo ncu=$?
ncu -i /tmp/p8.ncu-rep --page source --csv --print-source sass > gpurun_out/src_p8.csv 2>/dev/null
ncu -i /tmp/p8.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/mix_p8.csv 2>/dev/null
ncu -i /tmp/p8.ncu-rep --page raw --csv > gpurun_out/raw_p8.csv 2>/dev/null
python profiles/src_top.py gpurun_out/src_p8.csv 40
python profiles/line_hot.py gpurun_out/mix_p8.csv 40
