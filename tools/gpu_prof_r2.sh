#!/bin/bash
# round 2 profiles: per-tag DRAM bytes + binding unit (NVTX-renamed ncu launch lists) for
# C5 (rank-0 batch 0, eager) and C4 (one layer); ncu --set full of the C5 top kernels
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
DR_NVTX=1 DR_NO_GRAPH=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 200 --csv --log-file gpurun_out/nvtx_c5.csv python tools/c5_step.py 3 > /dev/null 2>&1; echo c5=$?
DR_NVTX=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 150 --csv --log-file gpurun_out/nvtx_c4.csv python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo c4=$?
python profiles/bounds.py gpurun_out/nvtx_c5.csv C5 > gpurun_out/bounds_c5.txt; python profiles/bounds.py gpurun_out/nvtx_c4.csv C4 > gpurun_out/bounds_c4.txt
cat gpurun_out/bounds_c5.txt | cut -c1-200
cp profiles/ncu_bounds.json profiles/ncu_traffic.json gpurun_out/
DR_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tc2_rows_kernel|tc2_reduce_kernel|tspmm_kernel" -s 0 -c 12 -o /tmp/full_c5 python tools/c5_step.py 1 > /dev/null 2>&1; echo full=$?
ncu -i /tmp/full_c5.ncu-rep --page raw --csv > gpurun_out/full_c5_raw.csv 2>/dev/null
ncu -i /tmp/full_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/full_c5_src.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/full_c5_raw.csv | cut -c1-250
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python -c "import json;j=json.load(open('gpurun_out/bench_default.json'));print(j['value'],j['ms_per_step'],j['roofline'],j['c4']['spmm_gate'])"
