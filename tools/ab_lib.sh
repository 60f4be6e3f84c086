# A/B of two libdr builds (abtmp/libdr_base.so, abtmp/libdr_new.so): GPU tests on the
# new one, then alternating C2 step / C4 layer bench lines with per-kernel means.
mkdir -p gpurun_out
L=paper_2508_16769_b200/libdr.so
cp abtmp/libdr_new.so $L
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for V in base new base new; do
cp abtmp/libdr_$V.so $L
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2> /dev/null
timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2> /dev/null
python - $V <<'PY'
import json, sys
j2 = json.load(open('gpurun_out/b2.json')); j4 = json.load(open('gpurun_out/b4.json'))
t = lambda j, p: {k: v['mean_ms'] for k, v in j['kernels'].items() if p in k}
print(sys.argv[1], 'C2', j2['value'], 'C4', j4['value'], t(j2, 'spmm_bwd.L1.cell'), t(j4, 'spmm_bwd.cell'))
PY
done
cp abtmp/libdr_new.so $L
