#!/bin/bash
mkdir -p gpurun_out
python tools/chain_prof.py 20 > gpurun_out/chainprof.txt 2>&1
DR_TC2_DEBUG=1 python tools/chain_prof.py 1 >> gpurun_out/chainprof.txt 2>&1
cat gpurun_out/chainprof.txt | grep -v "^\[tc2_rows" | tail -3
grep "tc2_rows" gpurun_out/chainprof.txt | sort | uniq -c | sort -rn | head -12 | cut -c1-400
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc2_rows_kernel -c 4 -o /tmp/chain python tools/chain_prof.py 1 > /dev/null 2>&1
ncu -i /tmp/chain.ncu-rep --page raw --csv > gpurun_out/chain_raw.csv 2>/dev/null
ncu -i /tmp/chain.ncu-rep --page source --csv --print-source sass > gpurun_out/chain_src.csv 2>/dev/null
cp /tmp/chain.ncu-rep gpurun_out/ 2>/dev/null
python profiles/ncu_table.py gpurun_out/chain_raw.csv | cut -c1-250
