"""NEXT-2 timing (DESIGN reading Q26): per relation, the sparse path
D-ReLU -> SpMM fwd -> SSpMM bwd (dX) with a uniform k (dr_drelu_topk + dr_spmm_fwd/bwd,
tensor-core tiled near where it applies) against the value-sorted D-ReLU + per-
destination-degree K schedule (dr_drelu_topk_sorted + dr_spmm_fwd_ng/bwd_ng, SIMT),
CUDA events, L2 flushed, median of 10. Also the fraction of (edge, pair) products the
schedule keeps. Prints one JSON object.  usage: python tools/ng_time.py [C2|C4 ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr
from gen import make_config

RELS = ("near", "pins", "pinned")


def timed(fn, flush, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)


out = {}
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for cfg in (sys.argv[1:] or ["C2", "C4"]):
    d = make_config(cfg)
    D, k = d.meta["D"], d.meta["k"]
    g = dr.Graph.from_design(d)
    xs = {"cell": torch.as_tensor(d.x_cell).cuda(), "net": torch.as_tensor(d.x_net).cuda()}
    scheds = {"k/2@8,k/4@32": ((8, 32), (k, k // 2, k // 4)),
              "k/2@16,k/4@64": ((16, 64), (k, k // 2, k // 4)),
              "uniform": ((8, 32), (k, k, k))}
    res = {}
    for rel in RELS:
        ptr, col, nd, ns = d.rel(rel)
        x = xs["net" if rel == "pinned" else "cell"]
        if x.shape[1] != D:
            x = torch.randn(ns, D, device="cuda")
        dz = torch.randn(nd, D, device="cuda")
        z = torch.empty(nd, D, device="cuda")
        dx = torch.empty(ns, D, device="cuda")
        deg = np.diff(ptr)

        v0, i0 = dr.drelu_topk(x, k)
        vs, is_ = dr.drelu_topk_sorted(x, k)
        r = {"plain": {
            "drelu": timed(lambda: dr.drelu_topk(x, k, out=(v0, i0)), flush),
            "fwd": timed(lambda: dr.spmm_fwd(g, rel, v0, i0, D, out=z), flush),
            "bwd": timed(lambda: dr.spmm_bwd(g, rel, dz, v0, i0, D, want_g=False, want_dx=True,
                                             dx_out=dx), flush)},
            "drelu_sorted": timed(lambda: dr.drelu_topk_sorted(x, k, out=(vs, is_)), flush)}
        for name, (thr, kb) in scheds.items():
            plan = dr.NgPlan(g, rel, thr, kb)
            K = np.where(deg <= thr[0], kb[0], np.where(deg <= thr[1], kb[1], kb[2]))
            r[name] = {
                "fwd": timed(lambda: dr.spmm_fwd_ng(plan, vs, is_, D, out=z), flush),
                "bwd": timed(lambda: dr.spmm_bwd_ng(plan, dz, vs, is_, D, want_g=False,
                                                    want_dx=True, dx_out=dx), flush),
                "pair_frac": round(float((K * deg).sum()) / max(1, k * deg.sum()), 4)}
        res[rel] = r
    out[cfg] = {"D": D, "k": k, "rels": res}
print(json.dumps(out))
