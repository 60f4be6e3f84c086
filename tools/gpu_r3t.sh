#!/bin/bash
mkdir -p gpurun_out
DR_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tc2_rows_kernel<\(int\)-1" -s 0 -c 1 -o /tmp/hd python tools/c5_step.py 1 > gpurun_out/ncu_hd.log 2>&1; echo ncu=$?
ncu -i /tmp/hd.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/mix_hd.csv 2>/dev/null
ncu -i /tmp/hd.ncu-rep --page source --csv --print-source sass > gpurun_out/src_hd.csv 2>/dev/null
python profiles/line_hot.py gpurun_out/mix_hd.csv 40
