#!/bin/bash
# ncu --set full captures of the tcgen05 dense kernels and the SSpMM on C2 (bench step).
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_reduce_kernel -s 6 -c 1 -o gpurun_out/prof_tc_reduce_c2 $B > gpurun_out/prof1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_rows_kernel -s 8 -c 2 -o gpurun_out/prof_tc_rows_c2 $B > gpurun_out/prof2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_bwd_kernel -s 6 -c 2 -o gpurun_out/prof_spmm_bwd_c4 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof3.log 2>&1
ls -la gpurun_out
