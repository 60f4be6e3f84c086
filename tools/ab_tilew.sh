# tiled SpMM CTA work split: chunk-balanced (W=0) vs chunks + W per tile
mkdir -p gpurun_out
for W in 0 2 4 8; do
DR_TS_TILE_W=$W DR_TS_DEBUG=1 timeout 300 python profiles/spmm_ab.py C2 default > gpurun_out/dbg_w$W.txt 2>&1
echo "W=$W"; grep "tspmm fwd\] max" gpurun_out/dbg_w$W.txt | head -1; grep "tspmm fwd D=" gpurun_out/dbg_w$W.txt | head -1 | cut -c1-80
DR_TS_TILE_W=$W timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/b2.json'));k=j['kernels'];print('W=$W C2',j['value'],k['spmm_fwd.L0.near']['mean_ms'],k['spmm_bwd.L1.cell']['mean_ms'])"
DR_TS_TILE_W=$W timeout 600 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2>/dev/null
python -c "import json;j=json.load(open('gpurun_out/b4.json'));k=j['kernels'];print('W=$W C4',j['value'],k['spmm_fwd.near']['mean_ms'],k['spmm_bwd.cell']['mean_ms'])"
done
