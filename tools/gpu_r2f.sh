#!/bin/bash
# C4 per-tag DRAM bytes / binding unit without the identity run mixed in; compute-sanitizer
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
DR_NVTX=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 100 --csv --log-file gpurun_out/nvtx_c4.csv python tools/c4_layer.py 2 > /dev/null 2>&1; echo c4=$?
DR_NVTX=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 100 --csv --log-file gpurun_out/nvtx_c4i.csv python tools/c4_layer.py 2 identity > /dev/null 2>&1; echo c4i=$?
python profiles/bounds.py gpurun_out/nvtx_c4.csv C4 > gpurun_out/bounds_c4.txt; python profiles/bounds.py gpurun_out/nvtx_c4i.csv C4-identity > gpurun_out/bounds_c4i.txt
cp profiles/ncu_bounds.json profiles/ncu_traffic.json gpurun_out/
cat gpurun_out/bounds_c4.txt | cut -c1-160
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1; echo $tool=$?; tail -3 gpurun_out/sanitize_$tool.log
done
