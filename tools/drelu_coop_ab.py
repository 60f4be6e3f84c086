"""A/B of the cooperative thread-per-row D-ReLU (knob drelu_coop: 0 = the default
kernel per shape, T = 2 / 4 lanes per row): CUDA events, L2 flushed, median of
20; every variant's output compared bit for bit with the default one. (Round 2
also measured a chunked thread-per-row variant here -- 1.6-4x slower, removed;
profiles/r02/ab_drelu_tpc.json.)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr

flush = torch.empty(256 << 20, device="cuda")
out = {}
for n, D, k in [(1_000_000, 128, 16), (700_000, 128, 16), (1_000_000, 128, 8), (100_000, 64, 8),
                (66_600, 64, 8), (300_000, 64, 16)]:
    x = torch.randn(n, D, device="cuda")
    x[:1000] = torch.randint(-2, 3, (1000, D), device="cuda").float()     # ties
    x[1000:1100] = 0.5
    ref = None
    row = {}
    for mode in (0, 1, 2, 4, -2):
        dr.debug_set("drelu_coop", mode)
        ts = []
        for it in range(23):
            flush.zero_()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            v, i = dr.drelu_topk(x, k)
            b.record()
            b.synchronize()
            if it >= 3:
                ts.append(a.elapsed_time(b))
        if ref is None:
            ref = (v.clone(), i.clone())
        same = bool(torch.equal(v, ref[0]) and torch.equal(i, ref[1]))
        ms = float(np.median(ts))
        row[f"coop{mode}"] = {"ms": round(ms, 4), "gbs": round(n * (D * 4 + 5 * k) / ms / 1e6, 1),
                              "bitexact_vs_default": same}
    dr.debug_set("drelu_coop", -2)
    out[f"{n}x{D} k{k}"] = row
print(json.dumps(out, indent=1))
