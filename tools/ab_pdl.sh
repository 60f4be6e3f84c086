mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for i in 1 2; do for P in 1 0; do
DR_PDL=$P timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_pdl$P.json 2> gpurun_out/bench_c2.err
python -c "import json;j=json.load(open('gpurun_out/bench_c2_pdl$P.json'));print('C2 PDL=$P',j['value'],j['ms_per_step'],j['e2e']['value'])"
done; done
for P in 1 0; do
DR_PDL=$P timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_pdl$P.json 2> gpurun_out/bench_c4.err
python -c "import json;j=json.load(open('gpurun_out/bench_c4_pdl$P.json'));print('C4 PDL=$P',j['value'],j['ms_per_step'])"
done
