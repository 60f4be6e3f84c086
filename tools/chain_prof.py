"""Fused next-layer D-ReLU (row a5) vs projection + standalone D-ReLU on one C5
batch: python tools/chain_prof.py [reps] [knob=value ...]. Prints CUDA-event
times of layer 1's forward in both forms (tc2_debug=1 adds role timers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2508_16769_b200 as dr
from gen import make_params
from gen.circuit import make_c5_set

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    dr.debug_set(k, int(v))
batches, _ = bench.c5_schedule(1, 4)
ids = batches[0][0]
d = bench.c5_batch_design(ids, make_c5_set(bench.C5_DESIGNS, only=ids))
g = dr.Graph.from_design(d)
D, k = 64, 8
P = make_params(D, D, D, 2, seed=7)
W = [{kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith(f"l{l}.")}
     for l in range(2)]
L1, L2 = dr.Layer(W[0], D, D, D, k, k), dr.Layer(W[1], D, D, D, k, k)
xc, xn = torch.as_tensor(d.x_cell).cuda(), torch.as_tensor(d.x_net).cuda()
t1 = torch.empty(L1.tape_bytes(g), dtype=torch.uint8, device="cuda")
t2 = torch.empty(L2.tape_bytes(g), dtype=torch.uint8, device="cuda")


def timeit(f):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


fused = lambda: dr.heteroconv_fwd_chain(g, L1, xc, xn, next_layer=L2, next_tape=t2, tape=t1,
                                        flags=dr.DR_FWD_Y_SCRATCH)


def plain():
    yc, yn, _ = dr.heteroconv_fwd(g, L1, xc, xn, tape=t1)
    dr.drelu_topk(yc, k)
    dr.drelu_topk(yn, k)


print(f"C5 batch {d.n_cell} cells: fused {timeit(fused):.4f} ms, plain+drelu {timeit(plain):.4f} ms")
