#!/bin/bash
# A/B of the SpMM processing order (degree vs locality) on C2 and C4.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
timeout 900 python profiles/spmm_ab.py C4 DR_ORDER=degree DR_ORDER=locality DR_ORDER=locality,DR_WARP_ROW_DEG=64 > gpurun_out/ab_order_c4.txt 2>&1
timeout 600 python profiles/spmm_ab.py C2 DR_ORDER=degree DR_ORDER=locality > gpurun_out/ab_order_c2.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
