"""A/B of the D-ReLU kernels (thread-per-row networks vs warp-per-row
extraction) at the C2 / C4 / C5 shapes: CUDA events, L2 flushed before each
launch, median of 20. Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr

flush = torch.empty(256 << 20, device="cuda")     # 1 GB: the host enqueues the timed launch meanwhile
out = {}
for n, D, k in [(100_000, 64, 8), (66_600, 64, 8), (1_000_000, 128, 16), (700_000, 128, 16),
                (300_000, 64, 16), (300_000, 64, 32)]:
    x = torch.randn(n, D, device="cuda")
    ov = torch.empty(n, k, device="cuda")
    oi = torch.empty(n, k, device="cuda", dtype=torch.uint8)
    row = {}
    for mode in (0, 2):
        dr.debug_set("drelu_tpr", mode)
        ts = []
        for it in range(23):
            flush.zero_()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            dr.drelu_topk(x, k, out=(ov, oi))
            b.record()
            b.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        row["tpr" if mode else "warp"] = {"ms": round(ms, 4),
                                          "gbs": round(n * (D * 4 + 5 * k) / ms / 1e6, 1)}
    dr.debug_set("drelu_tpr", 1)
    out[f"{n}x{D} k{k}"] = row
print(json.dumps(out))
