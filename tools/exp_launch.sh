#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
for E in "X=0" "DR_EXP_SKIP_PACK=1" "DR_EXP_SKIP_PARTS=1" "DR_EXP_SKIP_PACK=1 DR_EXP_SKIP_PARTS=1"; do
  env $E timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/e.json 2>/dev/null
  python -c "import json; j=json.load(open('gpurun_out/e.json')); print('$E', j['ms_per_step'], j['value'])"
done
