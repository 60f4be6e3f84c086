"""One C5 training batch (rank 0, batch 0 of bench.py's schedule) through
dr_train_step, for profilers: python tools/c5_step.py [steps] [knob=value ...]
Runs 3 eager warm-up steps, then `steps` steps (eager when no_graph=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2508_16769_b200 as dr
from gen import make_params
from gen.circuit import make_c5_set

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    dr.debug_set(k, int(v))
batches, _ = bench.c5_schedule(1, 4)
ids = batches[0][0]
designs = make_c5_set(bench.C5_DESIGNS, only=ids)
d = bench.c5_batch_design(ids, designs)
g = dr.Graph.from_design(d)
P = make_params(64, 64, 64, 2, seed=7)
flat = torch.as_tensor(dr.flatten_params(P, 2)).cuda()
tr = dr.Trainer(flat, 2, 64, 64, 64, 8, 8)
xc, xn, y = (torch.as_tensor(a).cuda() for a in (d.x_cell, d.x_net, d.labels))
for _ in range(3):
    tr.step(g, xc, xn, y)
torch.cuda.synchronize()
print(f"C5 batch: {d.n_cell} cells, {d.n_net} nets, nnz {d.nnz()}", file=sys.stderr)
for _ in range(steps):
    tr.step(g, xc, xn, y, sync=False)
torch.cuda.synchronize()
