#!/bin/bash
# tc2 parity tests, then ncu --set full of the tc2 row / reduce GEMMs in one C4 layer fwd+bwd.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "heteroconv or dense or train" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 300 python profiles/spmm_ab.py C4 default > gpurun_out/ab_c4.txt 2>&1
B="python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_rows_kernel -s 15 -c 5 -o gpurun_out/prof_tc2_rows_c4 $B > gpurun_out/p1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_reduce_kernel -s 9 -c 3 -o gpurun_out/prof_tc2_reduce_c4 $B > gpurun_out/p2.log 2>&1
ls gpurun_out
