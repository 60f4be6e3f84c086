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
# f4: peer-memory shard exchange and the sharded layer, 2 virtual ranks
W = 2
cp, _ = dr.shard_plan(*d.rel("near")[:2], d.rel("near")[3], W)
npart, _ = dr.shard_plan(*d.rel("pins")[:2], d.rel("pins")[3], W)
lays = []
for r in range(W):
    sn = dr.Shard.from_design(d, "near", W, r, dst_part=cp, src_part=cp)
    sp = dr.Shard.from_design(d, "pins", W, r, dst_part=npart, src_part=cp)
    sq = dr.Shard.from_design(d, "pinned", W, r, dst_part=cp, src_part=npart)
    lays.append((sn, sp, sq, dr.ShardLayer(sn, sp, sq)))
mc, mn = lays[0][0].max_src, lays[0][2].max_src
pc, pn = [], []
for r in range(W):
    xl = torch.zeros((mc, D), device="cuda")
    xl[:int(cp[r + 1] - cp[r])] = xc[int(cp[r]):int(cp[r + 1])]
    pc.append(dr.drelu_topk(xl, k))
    xl = torch.zeros((mn, D), device="cuda")
    xl[:int(npart[r + 1] - npart[r])] = xn[int(npart[r]):int(npart[r + 1])]
    pn.append(dr.drelu_topk(xl, k))
outs = [l[3].fwd(L1, pc, pn) for l in lays]
ibc = [torch.zeros((2, W, mc, k), device="cuda") for _ in range(W)]
ibn = [torch.zeros((W, mn, k), device="cuda") for _ in range(W)]
for r, l in enumerate(lays):
    l[3].bwd(L1, outs[r][2], torch.randn_like(outs[r][0]), torch.randn_like(outs[r][1]), pc, pn, ibc, ibn)
for r, l in enumerate(lays):
    l[3].dx(L1, outs[r][2], pc, pn, ibc[r], ibn[r])
    l[0].spmm_fwd_peer(pc, D, k)
torch.cuda.synchronize()
print("sanitize shard case done", file=sys.stderr)
