mkdir -p gpurun_out
DR_TC2_DEBUG=1 timeout 600 python profiles/spmm_ab.py C2 default > gpurun_out/dbg_tc2_c2.txt 2>&1
grep -h "tc2_rows\|tc2_reduce" gpurun_out/dbg_tc2_c2.txt | sort | uniq | awk '!seen[substr($0,1,70)]++' | head -20
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/bench_c2.json'))
print(j['value'], j['ms_per_step'], j['e2e'], j['roofline'])
ks=j['kernels']; tot=sum(v['total_ms'] for v in ks.values())
for t,v in sorted(ks.items(), key=lambda x:-x[1]['total_ms'])[:30]: print('  %-24s %8.4f ms  %5.1f%%  gbs=%s'%(t,v['mean_ms'],100*v['total_ms']/tot,v['gbs']))
print(' sum kernels per step', round(tot/j['steps'],4))
PY
