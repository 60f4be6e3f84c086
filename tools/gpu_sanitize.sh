#!/bin/bash
mkdir -p gpurun_out
python tools/sanitize_case.py 2>&1 | tail -2
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1; echo $tool=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" gpurun_out/sanitize_$tool.log | tail -2
done
