"""A/B of one libdr knob on one design: per-kernel times of one HeteroConv layer
fwd+bwd (eager, single stream, per-launch CUDA events) and the 3-stream wall
time. python tools/ab_knob.py C4|C2|C5 knob v1 v2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2508_16769_b200 as dr
from gen import make_config, make_params

wl = sys.argv[1]
name = sys.argv[2]
vals = [int(v) for v in sys.argv[3:]]
if wl == "C5":
    from gen.circuit import make_c5_set
    b, _ = bench.c5_schedule(1, 4)
    d = bench.c5_batch_design(b[0][0], make_c5_set(bench.C5_DESIGNS, only=b[0][0]))
    D, k = 64, 8
else:
    d = make_config(wl)
    D, k = (128, 16) if wl == "C4" else (64, 8)
P = make_params(D, D, D, 1, seed=7)
W = {kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith("l0.")}
L = dr.Layer(W, D, D, D, k, k)
xc, xn = torch.as_tensor(d.x_cell).cuda(), torch.as_tensor(d.x_net).cuda()
dyc = torch.randn(d.n_cell, D, device="cuda")
dyn = torch.randn(d.n_net, D, device="cuda")
flush = torch.empty(64 << 20, device="cuda")
for v in vals:
    dr.debug_set(name, v)
    g = dr.Graph.from_design(d)
    tape = torch.empty(L.tape_bytes(g), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        dr.heteroconv_fwd(g, L, xc, xn, tape=tape)
        dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)
    torch.cuda.synchronize()
    dr.profile_begin()
    for _ in range(5):
        flush.zero_()
        dr.heteroconv_fwd(g, L, xc, xn, tape=tape)
        dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)
    torch.cuda.synchronize()
    prof = dr.profile_end()
    sp = {t: round(tot / n * 1e3, 1) for t, (n, tot, mx) in prof.items()}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0.record()
        dr.heteroconv_fwd(g, L, xc, xn, tape=tape)
        dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{wl} {name}={v}: wall {sorted(ts)[5] * 1e3:.1f} us, kernel sum {sum(sp.values()):.1f} us",
          sp, flush=True)
    g.close()
