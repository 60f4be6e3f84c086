#!/bin/bash
# Round-end style check: build + smoke, GPU tests, C2/C4 bench lines (with CPU
# baseline on C2), ncu launch lists with per-tag DRAM bytes (NVTX-renamed kernels).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
DR_NVTX=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 150 --csv --log-file gpurun_out/traffic_c4.csv python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
DR_NVTX=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --metrics $M --clock-control none -c 150 --csv --log-file gpurun_out/traffic_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python profiles/traffic.py gpurun_out/traffic_c4.csv C4 > gpurun_out/traffic_c4.txt; python profiles/traffic.py gpurun_out/traffic_c2.csv C2 > gpurun_out/traffic_c2.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench4=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --workload C4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
head -c 600 gpurun_out/bench_c2.json; echo; head -c 600 gpurun_out/bench_c4.json
# ncu --set full of the C2 dominant kernels (tspmm bwd, spmm_fwd near) and the C4 one (tc2 rows proj.cell)
timeout 900 ncu --set full --clock-control none -k regex:tspmm -c 2 -o /tmp/full_ts_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i /tmp/full_ts_c2.ncu-rep --page raw --csv > gpurun_out/full_ts_c2_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:tc2_rows -s 1 -c 1 -o /tmp/full_proj_c4 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i /tmp/full_proj_c4.ncu-rep --page raw --csv > gpurun_out/full_proj_c4_raw.csv 2>/dev/null
python profiles/ncu_table.py gpurun_out/full_ts_c2_raw.csv | cut -c1-200; python profiles/ncu_table.py gpurun_out/full_proj_c4_raw.csv | cut -c1-200
