# SIMT forward sub-row CTAs A/B (the DR_SUB_CTAS knob was an experiment, since removed; results in profiles/r01/ab_sub_ctas.txt)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ng.py -x -q -k "spmm or heteroconv or ng" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for C in 0 1184 592 2368 0 1184; do
DR_SUB_CTAS=$C timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/b4.json'));k=j['kernels'];print('cap=$C C4',j['value'],k['spmm_fwd.pins']['mean_ms'],k['spmm_fwd.pinned']['mean_ms'])"
DR_SUB_CTAS=$C timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/b2.json'));k=j['kernels'];print('cap=$C C2',j['value'],k['spmm_fwd.L0.pins']['mean_ms'],k['spmm_fwd.L0.pinned']['mean_ms'])"
done
