#!/bin/bash
# ncu --set full of the tc2 row / reduce GEMMs in one C4 layer fwd+bwd.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
B="python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_rows_kernel -s 15 -c 5 -o gpurun_out/prof_tc2_rows_c4 $B > gpurun_out/p1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_reduce_kernel -s 15 -c 5 -o gpurun_out/prof_tc2_reduce_c4 $B > gpurun_out/p2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k dense > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
