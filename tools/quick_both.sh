mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tspmm.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edgek.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/b2.json'));k=j['kernels'];print('C2',j['value'],k['spmm_fwd.L0.near']['mean_ms'],k['spmm_bwd.L1.cell']['mean_ms'])"
timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/b4.json'));k=j['kernels'];print('C4',j['value'],k['spmm_fwd.near']['mean_ms'],k['spmm_bwd.cell']['mean_ms'],j['spmm_gate']['frac'])"
done
