# e2e with the NUMA-local host binding (bench.py), three runs, plus the NUMA topology.
mkdir -p gpurun_out
nvidia-smi topo -m 2>/dev/null | head -5
python - <<'PY'
import sys; sys.path.insert(0, '.')
import bench, torch
print("gpu-local cpus:", sorted(bench.gpu_local_cpus(0) or [])[:8], "...", len(bench.gpu_local_cpus(0) or []))
PY
for i in 1 2 3; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python -c "import json;j=json.load(open('gpurun_out/bench_c2.json'));print('C2',j['value'],j['ms_per_step'],j['e2e'])"
done
