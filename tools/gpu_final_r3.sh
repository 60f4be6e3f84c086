#!/bin/bash
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
# round 2 (session 3) final: per-tag DRAM bytes / binding units (C5, C4, C4-identity) with the final code,
# ncu launch lists of the default bench, ncu --set full of the top kernels, default bench line
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
DR_NVTX=1 DR_NO_GRAPH=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 200 --csv --log-file gpurun_out/nvtx_c5.csv python tools/c5_step.py 3 > /dev/null 2>&1; echo c5=$?
DR_NVTX=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 100 --csv --log-file gpurun_out/nvtx_c4.csv python tools/c4_layer.py 2 > /dev/null 2>&1; echo c4=$?
DR_NVTX=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 100 --csv --log-file gpurun_out/nvtx_c4i.csv python tools/c4_layer.py 2 identity > /dev/null 2>&1; echo c4i=$?
python profiles/bounds.py gpurun_out/nvtx_c5.csv C5 > gpurun_out/bounds_c5.txt
python profiles/bounds.py gpurun_out/nvtx_c4.csv C4 > gpurun_out/bounds_c4.txt
python profiles/bounds.py gpurun_out/nvtx_c4i.csv C4-identity > gpurun_out/bounds_c4i.txt
cp profiles/ncu_bounds.json profiles/ncu_traffic.json gpurun_out/
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c4 > /dev/null 2>&1; echo l5=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c4.csv python tools/c4_layer.py 2 > /dev/null 2>&1; echo l4=$?
DR_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tc2_rows_kernel|tspmm_kernel|tc2_reduce_kernel|drelu" -c 14 -o /tmp/full_c5 python tools/c5_step.py 1 > /dev/null 2>&1; echo f5=$?
ncu -i /tmp/full_c5.ncu-rep --page raw --csv > gpurun_out/full_c5_raw.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/full_c5_raw.csv > gpurun_out/ncu_full_c5.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tspmm_kernel|spmm_bwd_kernel|spmm_fwd_kernel|tc2_rows_kernel" -c 10 -o /tmp/full_c4 python tools/c4_layer.py 1 > /dev/null 2>&1; echo f4=$?
ncu -i /tmp/full_c4.ncu-rep --page raw --csv > gpurun_out/full_c4_raw.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/full_c4_raw.csv > gpurun_out/ncu_full_c4.txt
cut -c1-200 gpurun_out/ncu_full_c5.txt; cut -c1-200 gpurun_out/ncu_full_c4.txt
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref=$?
python -c "import json;j=json.load(open('gpurun_out/bench_default.json'));print(j['value'],j['ms_per_step'],j['e2e']['value'],j['roofline']['kernel'],j['roofline']['frac'],j['c4']['ms_per_iter'],j['c4']['spmm_gate']['frac'],j['c4']['spmm_gate'].get('dram_frac'))"
head -c 600 gpurun_out/bench_reference.json
