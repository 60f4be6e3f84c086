"""Role timers (DR_TC2_DEBUG / DR_TS_DEBUG) of one C4 layer fwd+bwd, eager."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_16769_b200 as dr
from gen import make_config, make_params

d = make_config("C4")
g = dr.Graph.from_design(d)
D, k = 128, 16
P = make_params(D, D, D, 1, seed=7)
W = {kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith("l0.")}
L = dr.Layer(W, D, D, D, k, k)
tape = torch.empty(L.tape_bytes(g), dtype=torch.uint8, device="cuda")
xc, xn = torch.as_tensor(d.x_cell).cuda(), torch.as_tensor(d.x_net).cuda()
dyc = torch.randn(d.n_cell, D, device="cuda")
dyn = torch.randn(d.n_net, D, device="cuda")
for it in range(2):
    if it == 1:
        dr.debug_set("tc2_debug", 1)
        dr.debug_set("ts_debug", 1)
    dr.heteroconv_fwd(g, L, xc, xn, tape=tape, flags=dr.DR_FWD_SEQUENTIAL)
    dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True, flags=dr.DR_FWD_SEQUENTIAL)
    torch.cuda.synchronize()
