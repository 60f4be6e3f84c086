#!/bin/bash
# ncu --set full of the SpMM forward (near) and the cell-source SSpMM on C4.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
B="python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_fwd_kernel -s 9 -c 1 -o gpurun_out/prof_spmm_fwd_c4 $B > gpurun_out/p1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bwd_kernel -s 6 -c 1 -o gpurun_out/prof_spmm_bwd_c4 $B > gpurun_out/p2.log 2>&1
ls gpurun_out
