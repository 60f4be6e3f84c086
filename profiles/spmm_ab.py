"""Isolated SpMM timings (CUDA events, L2 flushed) on one config under several
graph-creation settings (env assignments such as DR_ORDER=degree,
DR_ORDER=locality, DR_WARP_ROW_DEG=64); used to pick the processing order and
the warp-row class boundary. Also times one fused HeteroConv layer fwd+bwd.
usage: python profiles/spmm_ab.py C4 [setting ...]   (setting "default" = no env)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr
from gen import make_config, make_params

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
settings = sys.argv[2:] or ["default"]
t0 = time.time()
d = make_config(cfg)
D, k = d.meta["D"], d.meta["k"]
print(f"generated {cfg} in {time.time() - t0:.1f}s", file=sys.stderr)
xc = torch.as_tensor(d.x_cell).cuda()
xn = torch.as_tensor(d.x_net).cuda()
hc = dr.drelu_topk(xc, k)
hn = dr.drelu_topk(xn, k)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
src = {"near": hc, "pins": hc, "pinned": hn}
nd = {"near": d.n_cell, "pins": d.n_net, "pinned": d.n_cell}
dz = {r: torch.randn(nd[r], D, device="cuda") for r in src}
nnz = d.nnz()
P = make_params(D, D, D, 1, seed=7)
W = {kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith("l0.")}
L = dr.Layer(W, D, D, D, k, k)
dyc = torch.randn(d.n_cell, D, device="cuda")
dyn = torch.randn(d.n_net, D, device="cuda")


def timeit(fn, reps=5):
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
    return float(np.median(ts))


for st in settings:
    for kk in ("DR_ORDER", "DR_WARP_ROW_DEG"):
        os.environ.pop(kk, None)
    if st != "default":
        for kv in st.split(","):
            kk, vv = kv.split("=")
            os.environ[kk] = vv
    t0 = time.time()
    g = dr.Graph.from_design(d)
    res = {"create_s": time.time() - t0}
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
    tape = torch.empty(L.tape_bytes(g), dtype=torch.uint8, device="cuda")
    res["layer.fwd"] = timeit(lambda: dr.heteroconv_fwd(g, L, xc, xn, tape=tape))
    res["layer.fwd_bwd"] = timeit(lambda: (dr.heteroconv_fwd(g, L, xc, xn, tape=tape),
                                           dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)))
    dr.profile_begin()
    for _ in range(3):
        flush.zero_()
        dr.heteroconv_fwd(g, L, xc, xn, tape=tape, flags=1)
        dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True, flags=1)
    torch.cuda.synchronize()
    prof = dr.profile_end()
    res["seq_kernels_ms"] = {t: round(v[1] / v[0], 4) for t, v in sorted(prof.items())}
    print(st, json.dumps({kk: (round(vv, 4) if isinstance(vv, float) else vv)
                          for kk, vv in res.items()}), flush=True)
    del g
