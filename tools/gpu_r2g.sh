#!/bin/bash
mkdir -p gpurun_out
DR_NO_GRAPH=1 python tools/c5_step.py 1 ts_debug=1 tc2_debug=1 > gpurun_out/roles_c5.txt 2>&1; grep "\[" gpurun_out/roles_c5.txt | tail -24 | cut -c1-330
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
