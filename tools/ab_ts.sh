# A/B of two libdr builds (abtmp/libdr_base.so vs abtmp/libdr_new.so): tests on the
# new one, then isolated SpMM timings and bench lines, alternating.
mkdir -p gpurun_out
L=paper_2508_16769_b200/libdr.so
cp abtmp/libdr_new.so $L
timeout 900 python -m pytest tests/test_gpu_tspmm.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for V in base new base new; do
cp abtmp/libdr_$V.so $L
for C in C2 C4; do
timeout 600 python profiles/spmm_ab.py $C default > gpurun_out/ab_$C.txt 2>&1
python - $C $V <<'PY'
import json,sys
for line in open('gpurun_out/ab_%s.txt'%sys.argv[1]):
    if line.startswith('default'):
        name, js = line.split(' ',1); j=json.loads(js); sk=j['seq_kernels_ms']
        print(sys.argv[2], sys.argv[1], 'layer', j['layer.fwd_bwd'], {k:v for k,v in sk.items() if 'spmm' in k})
PY
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "import json;j=json.load(open('gpurun_out/bench_c2.json'));print('$V C2',j['value'],j['ms_per_step'],j['roofline']['kernel'],j['roofline']['frac'])"
done
cp abtmp/libdr_new.so $L
