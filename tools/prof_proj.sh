# ncu source-level (SASS) hot spots of the C4 cell projection (tc2_rows_kernel, first launch)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_rows -c 1 \
  -o /tmp/full_proj python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/full_proj.log 2>&1
echo rc=$?
ncu -i /tmp/full_proj.ncu-rep --page source --csv --print-source sass > gpurun_out/full_proj_sass.csv 2>/dev/null
ncu -i /tmp/full_proj.ncu-rep --page source --csv --print-source cuda > gpurun_out/full_proj_src.csv 2>/dev/null
python profiles/sass_hot.py gpurun_out/full_proj_sass.csv 40
