# per-direction CTA split weights: forward DR_TS_TILE_W, backward DR_TS_TILE_W_BWD
mkdir -p gpurun_out
for WF in 0 1; do for WB in 2 3; do
DR_TS_TILE_W=$WF DR_TS_TILE_W_BWD=$WB timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/b2.json'));k=j['kernels'];print('WF=$WF WB=$WB C2',j['value'],k['spmm_fwd.L0.near']['mean_ms'],k['spmm_bwd.L1.cell']['mean_ms'])"
DR_TS_TILE_W=$WF DR_TS_TILE_W_BWD=$WB timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/b4.json'));k=j['kernels'];print('WF=$WF WB=$WB C4',j['value'],k['spmm_fwd.near']['mean_ms'],k['spmm_bwd.cell']['mean_ms'])"
done; done
