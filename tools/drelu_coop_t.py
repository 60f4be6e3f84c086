"""A/B: lanes per row (drelu_coop T = 1, 2, 4) of the cooperative D-ReLU at the C5
shapes; CUDA events, L2 flushed, median of 20."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr

flush = torch.empty(256 << 20, device="cuda")
for n, D, k in [(101044, 64, 8), (77676, 64, 8)]:
    x = torch.randn(n, D, device="cuda")
    ov = torch.empty(n, k, device="cuda")
    oi = torch.empty(n, k, device="cuda", dtype=torch.uint8)
    row = {}
    for T in (1, 2, 4):
        for roll in (0, 2):
            dr.debug_set("drelu_coop", T)
            dr.debug_set("tpr_stream", roll)
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
            row[f"T{T}r{roll}"] = round(float(np.median(ts)), 4)
    dr.debug_set("drelu_coop", -2)
    dr.debug_set("tpr_stream", 1)
    print(f"{n}x{D} k{k}", row, flush=True)
