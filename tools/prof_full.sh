#!/bin/bash
# ncu --set full of every hot kernel of one C4 layer fwd+bwd (first step) and of
# one C2 training step. The C4 report comes back whole (read here with
# `ncu -i ... --page raw --csv`); the C2 one is exported to CSV on the box.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
K='regex:drelu|spmm_fwd|spmm_bwd|tc2_rows_kernel|tc2_reduce_kernel|head_kernel'
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -c 15 \
  -o gpurun_out/full_c4 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_c4.log 2>&1
echo c4=$?
timeout 900 ncu --set full --clock-control none -k "$K" -c 20 \
  -o /tmp/full_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_c2.log 2>&1
echo c2=$?
ncu -i /tmp/full_c2.ncu-rep --page raw --csv > gpurun_out/full_c2_raw.csv 2>/dev/null
ls -la gpurun_out
