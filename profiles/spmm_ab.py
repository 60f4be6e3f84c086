"""Isolated SpMM timings (CUDA events, L2 flushed) on one config under several
settings of DR_WARP_ROW_DEG; used to pick the warp-row class boundary.
usage: python profiles/spmm_ab.py C4 [thresholds...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr
from gen import make_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
ths = [x for x in sys.argv[2:]] or ["default"]
t0 = time.time()
d = make_config(cfg)
D, k = d.meta["D"], d.meta["k"]
print(f"generated {cfg} in {time.time() - t0:.1f}s", file=sys.stderr)
g = dr.Graph.from_design(d)
xc = torch.as_tensor(d.x_cell).cuda()
xn = torch.as_tensor(d.x_net).cuda()
hc = dr.drelu_topk(xc, k)
hn = dr.drelu_topk(xn, k)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
src = {"near": hc, "pins": hc, "pinned": hn}
nd = {"near": d.n_cell, "pins": d.n_net, "pinned": d.n_cell}
dz = {r: torch.randn(nd[r], D, device="cuda") for r in src}
nnz = d.nnz()


def timeit(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


out = {}
for th in ths:
    if th == "default":
        os.environ.pop("DR_WARP_ROW_DEG", None)
    else:
        os.environ["DR_WARP_ROW_DEG"] = th
    res = {}
    for r in ("near", "pins", "pinned"):
        v, i = src[r]
        z = torch.empty(nd[r], D, device="cuda")
        res["fwd." + r] = timeit(lambda: dr.spmm_fwd(g, r, v, i, D, out=z))
        gk = torch.empty(v.shape, device="cuda")
        res["bwd." + r] = timeit(lambda: dr.spmm_bwd(g, r, dz[r], v, i, D, g_out=gk))
    fb = nnz["near"] * (4 + 5 * k) + d.n_cell * (4 + 4 * D)
    res["fwd.near.alg_GBs"] = fb / (res["fwd.near"] * 1e-3) / 1e9
    bb = nnz["near"] * (4 + 4 * k) + d.n_cell * (k + 4 * k)
    res["bwd.near.alg_GBs"] = bb / (res["bwd.near"] * 1e-3) / 1e9
    out[th] = res
    print(th, json.dumps({kk: round(vv, 4) for kk, vv in res.items()}))
