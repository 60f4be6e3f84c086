"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): a 2k-cell
C2-shaped design (tiled near path, hubs) through one layer fwd+bwd (plain and
chained with the fused next-layer D-ReLU) and two training steps, plus the
standalone D-ReLU / SpMM / SSpMM calls. python tools/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2508_16769_b200 as dr
from gen import make_config, make_params

d = make_config("C2", scale=0.02)
g = dr.Graph.from_design(d)
print("tiles", g.info()["tiles"], file=sys.stderr)
D, k = 64, 8
P = make_params(D, D, D, 2, seed=3)
W = [{kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith(f"l{l}.")}
     for l in range(2)]
L1, L2 = dr.Layer(W[0], D, D, D, k, k), dr.Layer(W[1], D, D, D, k, k)
xc, xn = torch.as_tensor(d.x_cell).cuda(), torch.as_tensor(d.x_net).cuda()
yc, yn, tape = dr.heteroconv_fwd(g, L1, xc, xn)
dr.heteroconv_bwd(g, L1, tape, torch.randn_like(yc), torch.randn_like(yn), need_dx=True)
yc2, yn2, t1, t2 = dr.heteroconv_fwd_chain(g, L1, xc, xn, next_layer=L2, flags=dr.DR_FWD_Y_SCRATCH)
dr.heteroconv_fwd_chain(g, L2, None, None, tape=t2, flags=dr.DR_FWD_INPUT_IN_TAPE)
val, idx = dr.drelu_topk(xc, k)
z = dr.spmm_fwd(g, dr.DR_NEAR, val, idx, D)
dr.spmm_bwd(g, dr.DR_NEAR, z, val, idx, D, want_dx=True)
flat = torch.as_tensor(dr.flatten_params(P, 2)).cuda()
tr = dr.Trainer(flat, 2, D, D, D, k, k)
for _ in range(3):                       # eager, captured, replayed
    tr.step(g, xc, xn, torch.as_tensor(d.labels).cuda())
torch.cuda.synchronize()
print("sanitize case done", file=sys.stderr)
