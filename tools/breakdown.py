"""SURVEY §8 f3 / paper §4.4 breakdown on CircuitNet-sized graphs:
(1) kernel savings: one HeteroConv layer fwd+bwd with the D-ReLU sparse
features (k) vs the dense-feature equivalent (k = D, every value kept) through
the same kernels; (2) parallel savings: the three relations on three streams vs
one stream (DR_FWD_SEQUENTIAL); (3) graph initialisation on 3 worker threads vs
1 (dr_graph_create n_threads, Alg. 1/2 stage 1, §3.4). Timing: CUDA events,
median of 20 (layer), wall clock median of 5 (init). Prints one JSON object.
usage: python tools/breakdown.py [C5|C2]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr
from gen import make_config, make_params
from gen.circuit import disjoint_union, make_c5_set

which = sys.argv[1] if len(sys.argv) > 1 else "C5"
if which == "C5":
    designs = make_c5_set(n_designs=4)
    d = disjoint_union(designs[0])      # one Mini-CircuitNet design: 2-4 graphs
    D, k = 64, 8
else:
    d = make_config(which)
    D, k = d.meta["D"], d.meta["k"]
g = dr.Graph.from_design(d)
xc = torch.as_tensor(d.x_cell).cuda()
xn = torch.as_tensor(d.x_net).cuda()
P = make_params(D, D, D, 1, seed=7)
W = {kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith("l0.")}
dyc = torch.randn(d.n_cell, D, device="cuda")
dyn = torch.randn(d.n_net, D, device="cuda")


def layer_ms(kk, flags):
    L = dr.Layer(W, D, D, D, kk, kk)
    tape = torch.empty(L.tape_bytes(g, flags), dtype=torch.uint8, device="cuda")

    def step():
        dr.heteroconv_fwd(g, L, xc, xn, tape=tape, flags=flags)
        dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True, flags=flags)

    for _ in range(3):
        step()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        step()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


SEQ = dr.DR_FWD_SEQUENTIAL
out = {"graph": which, "n_cell": d.n_cell, "n_net": d.n_net, "nnz": d.nnz(), "D": D, "k": k}
out["layer_ms"] = {"sparse_k_3streams": layer_ms(k, 0), "sparse_k_1stream": layer_ms(k, SEQ),
                   "dense_kD_3streams": layer_ms(D, 0), "dense_kD_1stream": layer_ms(D, SEQ)}
lm = out["layer_ms"]
out["kernel_saving"] = round(1 - lm["sparse_k_1stream"] / lm["dense_kD_1stream"], 4)
out["parallel_saving"] = round(1 - lm["sparse_k_3streams"] / lm["sparse_k_1stream"], 4)
init = {}
for nt in (1, 3):
    ts = []
    for _ in range(5):
        t = time.time()
        gg = dr.Graph.from_design(d, n_threads=nt)
        torch.cuda.synchronize()
        ts.append(time.time() - t)
        gg.close()
    init[f"threads_{nt}_ms"] = round(1e3 * float(np.median(ts)), 3)
out["graph_init"] = init
print(json.dumps(out))
