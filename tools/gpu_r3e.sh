#!/bin/bash
mkdir -p gpurun_out
DR_NO_GRAPH=1 DR_TC2_DEBUG=1 timeout 300 python tools/c5_step.py 1 2>&1 | grep "tc2_rows" | tail -10 | cut -c1-300
DR_NO_GRAPH=1 DR_TC2_DEBUG=1 timeout 300 ncu --metrics gpu__time_duration.sum --kernel-name-base demangled -k regex:tc2_rows --csv python tools/c5_step.py 1 2>&1 | grep -v "^==" | tail -12 | cut -c1-250
