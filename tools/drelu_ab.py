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
for n, D, k in [(100_000, 64, 4), (100_000, 64, 2), (100_000, 64, 8), (66_600, 64, 8), (1_000_000, 128, 16), (700_000, 128, 16),
                (300_000, 64, 16), (300_000, 64, 32)]:
    x = torch.randn(n, D, device="cuda")
    ov = torch.empty(n, k, device="cuda")
    oi = torch.empty(n, k, device="cuda", dtype=torch.uint8)
    row = {}
    modes = {"warp": dict(drelu_tpr=0), "tpr": dict(drelu_tpr=2, drelu_coop=0, tpr_stream=0),
             "tpr_stream": dict(drelu_tpr=2, drelu_coop=0, tpr_stream=2),
             "coop": dict(drelu_tpr=2, drelu_coop=2, tpr_stream=0),
             "coop_roll": dict(drelu_tpr=2, drelu_coop=2, tpr_stream=2), "default": {}}
    for name, kn in modes.items():
        base = dict(drelu_tpr=1, drelu_coop=-2, tpr_stream=1)
        base.update(kn)
        for kk, vv in base.items():
            dr.debug_set(kk, vv)
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
        row[name] = {"ms": round(ms, 4),
                                          "gbs": round(n * (D * 4 + 5 * k) / ms / 1e6, 1)}
    for kk, vv in dict(drelu_tpr=1, drelu_coop=-2, tpr_stream=1).items():
        dr.debug_set(kk, vv)
    out[f"{n}x{D} k{k}"] = row
print(json.dumps(out))
