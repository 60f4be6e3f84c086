#!/bin/bash
# refresh C5 per-tag DRAM bytes / binding units and the ncu full table with the final code (dual-B dW tag)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
DR_NVTX=1 DR_NO_GRAPH=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 200 --csv --log-file gpurun_out/nvtx_c5.csv python tools/c5_step.py 3 > /dev/null 2>&1; echo c5=$?
python profiles/bounds.py gpurun_out/nvtx_c5.csv C5 > gpurun_out/bounds_c5.txt
cp profiles/ncu_bounds.json profiles/ncu_traffic.json gpurun_out/
DR_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tc2_rows_kernel|tspmm_kernel|tc2_reduce_kernel|drelu" -c 14 -o /tmp/full_c5 python tools/c5_step.py 1 > /dev/null 2>&1; echo f5=$?
ncu -i /tmp/full_c5.ncu-rep --page raw --csv > gpurun_out/full_c5_raw.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/full_c5_raw.csv > gpurun_out/ncu_full_c5.txt
cut -c1-200 gpurun_out/ncu_full_c5.txt
timeout 600 python bench.py --no-cpu-baseline --no-c4 > gpurun_out/bench_after_traffic.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/bench_after_traffic.json'));print(j['value'],j['roofline'])"
