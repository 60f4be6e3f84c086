"""One C4 HeteroConv layer fwd+bwd (bench.py's C4 workload, same design, params
and inputs) for profilers: python tools/c4_layer.py [iters] [identity]
`identity` builds the graph with DR_GRAPH_ORDER_IDENTITY (bench.py's pure-DRAM
gate run). Eager calls on one stream when DR_FORCE_SEQUENTIAL=1 is set."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_16769_b200 as dr
from gen import make_config, make_params

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ident = len(sys.argv) > 2 and sys.argv[2] == "identity"
D, k = 128, 16
d = make_config("C4")
g = dr.Graph.from_design(d, flags=dr.DR_GRAPH_ORDER_IDENTITY if ident else 0)
P = make_params(D, D, D, 1, seed=7)
W = {kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith("l0.")}
L = dr.Layer(W, D, D, D, k, k)
tape = torch.empty(L.tape_bytes(g), dtype=torch.uint8, device="cuda")
xc, xn = torch.as_tensor(d.x_cell).cuda(), torch.as_tensor(d.x_net).cuda()
dyc = torch.randn(d.n_cell, D, device="cuda")
dyn = torch.randn(d.n_net, D, device="cuda")
for _ in range(iters):
    dr.heteroconv_fwd(g, L, xc, xn, tape=tape)
    dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)
torch.cuda.synchronize()
print("done", file=sys.stderr)
