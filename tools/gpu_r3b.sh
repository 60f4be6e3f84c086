#!/bin/bash
# C5 role timers of the tcgen05 kernels (eager step)
mkdir -p gpurun_out
DR_NO_GRAPH=1 DR_TC2_DEBUG=1 DR_TS_DEBUG=1 timeout 300 python tools/c5_step.py 1 > gpurun_out/roles_c5.txt 2>&1; echo roles=$?
tail -40 gpurun_out/roles_c5.txt | cut -c1-400
