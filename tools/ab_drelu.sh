# D-ReLU: successive-max extraction (default for k <= 32) vs the row-wise binary
# search (DR_DRELU_BS=1), isolated (CUDA events, L2 flushed) at C2 and C4 shapes.
mkdir -p gpurun_out
for BS in 0 1 0 1; do
DR_DRELU_BS=$BS timeout 300 python - <<'PY'
import os, torch, numpy as np, paper_2508_16769_b200 as dr
fl = torch.empty(64 * 1024 * 1024, device="cuda")
def t(fn, reps=10):
    fn(); ts = []
    for _ in range(reps):
        fl.zero_(); a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)
out = {}
for n, D, k in ((100000, 64, 8), (1000000, 128, 16), (300000, 64, 4), (300000, 64, 32)):
    x = torch.randn(n, D, device="cuda")
    v = torch.empty(n, k, device="cuda"); i = torch.empty(n, k, device="cuda", dtype=torch.uint8)
    out[f"{n}x{D} k={k}"] = t(lambda: dr.drelu_topk(x, k, out=(v, i)))
print("BS=" + os.environ.get("DR_DRELU_BS", "0"), out)
PY
done
