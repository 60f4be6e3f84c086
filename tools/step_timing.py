"""Per-step device times of the C5 training step under several enqueue schemes
(diagnosis of outlier steps in bench.py's timed loop). Prints, per scheme, the
steps slower than 0.7 ms and the host enqueue time of each such step."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2508_16769_b200 as dr
from gen import make_params
from gen.circuit import make_c5_set

batches, _ = bench.c5_schedule(1, 4)
S = len(batches)
mine = [batches[s][0] for s in range(S)]
need = sorted({i for b in mine for i in b})
designs = make_c5_set(bench.C5_DESIGNS, only=need, workers=8)
bd = [bench.c5_batch_design(b, designs) for b in mine]
graphs = [dr.Graph.from_design(x) for x in bd]
inputs = [tuple(torch.as_tensor(a).cuda() for a in (x.x_cell, x.x_net, x.labels)) for x in bd]
P = make_params(64, 64, 64, 2, seed=7)
flat = torch.as_tensor(dr.flatten_params(P, 2)).cuda()
tr = dr.Trainer(flat, 2, 64, 64, 64, 8, 8)
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
for s in range(S):
    for _ in range(2):
        tr.step(graphs[s], *inputs[s], sync=False)
torch.cuda.synchronize()


def run(name, n, chunk, sleep0, sleep_c, nogc):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    host = [0.0] * n
    if nogc:
        gc.collect()
        gc.disable()
    for c0 in range(0, n, chunk):
        torch.cuda.synchronize()
        sl = sleep0 if c0 == 0 else sleep_c
        if sl:
            torch.cuda._sleep(int(2e9 * sl))
        for i in range(c0, min(n, c0 + chunk)):
            t0 = time.perf_counter()
            flush.zero_()
            ev[i][0].record()
            tr.step(graphs[i % S], *inputs[i % S], sync=False)
            ev[i][1].record()
            host[i] = time.perf_counter() - t0
    torch.cuda.synchronize()
    gc.enable()
    per = [a.elapsed_time(b) for a, b in ev]
    slow = [(i, round(per[i], 3), round(host[i] * 1e3, 2)) for i in range(n) if per[i] > 0.7]
    hs = sorted(host)
    print(f"{name}: sum {sum(per):.2f} ms, median {sorted(per)[n // 2]:.3f}, host median "
          f"{hs[n // 2] * 1e3:.3f} ms max {hs[-1] * 1e3:.2f} ms; slow (i, ms, host ms): {slow}", flush=True)


for rep in range(2):
    run("plain", 100, 100, 0, 0, False)
    run("plain+lead", 100, 100, 0.2, 0, False)
    run("chunk16", 100, 16, 0.1, 0.1, True)
    run("plain+lead+nogc", 100, 100, 0.2, 0, True)
