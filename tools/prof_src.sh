#!/bin/bash
# source-level (SASS) stall profiles of several kernels in one C4 layer
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
B="python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline"
prof() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 -o /tmp/$1 $B > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/raw_$1.csv 2>/dev/null
}
prof dznear tc2_rows 2
prof drelu drelu 0
prof fwdpins spmm_fwd 0
prof bwdnet spmm_bwd 1
for f in dznear drelu fwdpins bwdnet; do python profiles/ncu_table.py gpurun_out/raw_$f.csv | tail -1 | cut -c1-200; done
