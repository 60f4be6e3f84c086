"""BASELINE configs[2]: CircuitNet-medium-shaped design (C3: 300k cells, 200k nets,
hidden 64), D-ReLU k sweep {8, 16, 32}: one HeteroConv layer fwd+bwd per k (CUDA
events, L2 flushed, median of 10), plus the per-relation K-profile (SURVEY §8 f1,
paper_2508_16769_b200.kprof) over k in {2, ..., 64}. Prints one JSON object.
usage: python tools/ksweep.py [C3|C2]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr
from gen import make_config, make_params
from paper_2508_16769_b200.kprof import kprofile

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
t0 = time.time()
d = make_config(cfg)
D = d.meta["D"]
g = dr.Graph.from_design(d)
xc = torch.as_tensor(d.x_cell).cuda()
xn = torch.as_tensor(d.x_net).cuda()
P = make_params(D, D, D, 1, seed=7)
W = {kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith("l0.")}
flush = torch.empty(64 * 1024 * 1024, device="cuda")
dyc = torch.randn(d.n_cell, D, device="cuda")
dyn = torch.randn(d.n_net, D, device="cuda")
out = {"config": cfg, "n_cell": d.n_cell, "n_net": d.n_net, "nnz": d.nnz(), "D": D,
       "layer_fwd_bwd_ms": {}}
for k in (8, 16, 32):
    L = dr.Layer(W, D, D, D, k, k)
    tape = torch.empty(L.tape_bytes(g), dtype=torch.uint8, device="cuda")

    def step():
        dr.heteroconv_fwd(g, L, xc, xn, tape=tape)
        dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)

    step()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        step()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    out["layer_fwd_bwd_ms"][k] = round(float(np.median(ts)), 4)
out["kprofile"] = kprofile(g, xc, xn, ks=(2, 4, 8, 16, 32, 64), reps=5)
out["wall_s"] = round(time.time() - t0, 1)
print(json.dumps(out))
