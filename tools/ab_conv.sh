# A/B of two libdr builds on the C2 step and C4 layer with per-kernel tables.
mkdir -p gpurun_out
L=paper_2508_16769_b200/libdr.so
cp abtmp/libdr_new.so $L
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tspmm.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for V in base new base new; do
cp abtmp/libdr_$V.so $L
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2> /dev/null
timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2> /dev/null
python - $V <<'PY'
import json, sys
j2 = json.load(open('gpurun_out/b2.json')); j4 = json.load(open('gpurun_out/b4.json'))
t = lambda j, p: {k: v['mean_ms'] for k, v in j['kernels'].items() if k.startswith(p)}
print(sys.argv[1], 'C2', j2['value'], 'C4', j4['value'], 'proj4', t(j4, 'tc_proj'), 'dz4', t(j4, 'tc_dz'), 'proj2', t(j2, 'tc_proj.L0'))
PY
done
cp abtmp/libdr_new.so $L
