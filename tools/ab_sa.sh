# C2 step vs the tiled SpMM's stage count (DR_TS_MAXSA): shared-memory footprint
# against cross-stream concurrency. (The DR_TS_MAXSA knob this needs was an experiment, since removed; results in profiles/r01/ab_tspmm_pipeline.txt.)
mkdir -p gpurun_out
for r in 1 2; do for SA in 4 3; do   # SA = 2 deadlocks (launch() now rejects it)
DR_TS_MAXSA=$SA timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "import json;j=json.load(open('gpurun_out/bench_c2.json'));k=j['kernels'];print('SA=$SA C2',j['value'],j['ms_per_step'],k['spmm_fwd.L0.near']['mean_ms'],k['spmm_bwd.L1.cell']['mean_ms'])"
done; done
