"""§8 f4 timing on one GPU: C4 (1M cells, D=128, k=16), one relation split over W
virtual ranks. Per W: the slowest rank's dr_shard_spmm_fwd + dr_shard_spmm_bwd time
(CUDA events, L2 flushed, median of 5) against the single-graph dr_spmm_fwd + bwd,
and the bytes each exchange moves per rank (CBSR allgather in, g reduce-scatter
out) against the dense-feature allgather it replaces. Prints one JSON object.
usage: python tools/shard_time.py [C4|C2] [spatial|shuffled] [rel ...]
(spatial: node ids in a locality order, so a rank's contiguous rows are a compact
region; DR_SHARD_TILES=1 gives near's blocks the tensor-core tiled forward)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_16769_b200 as dr
from gen import make_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
order = sys.argv[2] if len(sys.argv) > 2 else "shuffled"
rels = sys.argv[3:] or ["near", "pins", "pinned"]
d = make_config(cfg, order=order)
D, k = d.meta["D"], d.meta["k"]
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def timed(fn, reps=5):
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
    return round(float(np.median(ts)), 4)


g = dr.Graph.from_design(d)
out = {"config": cfg, "order": order, "D": D, "k": k, "rels": {}}
for rel in rels:
    ptr, col, nd, ns = d.rel(rel)
    X = torch.randn(ns, D, device="cuda")
    dZ = torch.randn(nd, D, device="cuda")
    v, i = dr.drelu_topk(X, k)
    z = torch.empty(nd, D, device="cuda")
    gk = torch.empty(ns, k, device="cuda")
    full = timed(lambda: (dr.spmm_fwd(g, rel, v, i, D, out=z),
                          dr.spmm_bwd(g, rel, dZ, v, i, D, g_out=gk)))
    r = {"single_graph_ms": full,
         "single_graph_fwd_ms": timed(lambda: dr.spmm_fwd(g, rel, v, i, D, out=z)),
         "single_graph_bwd_ms": timed(lambda: dr.spmm_bwd(g, rel, dZ, v, i, D, g_out=gk)),
         "world": {}}
    for W in (2, 4, 8):
        shards = [dr.Shard.from_design(d, rel, W, q) for q in range(W)]
        m = shards[0].max_src
        va = torch.zeros(W * m, k, device="cuda")
        ia = torch.zeros(W * m, k, device="cuda", dtype=torch.uint8)
        for q, sh in enumerate(shards):
            n = sh.src_end - sh.src_begin
            va[q * m:q * m + n] = v[sh.src_begin:sh.src_end]
            ia[q * m:q * m + n] = i[sh.src_begin:sh.src_end]
        per, pf, pb = [], [], []
        for sh in shards:
            zl = torch.empty(sh.dst_end - sh.dst_begin, D, device="cuda")
            gp = torch.empty(W * m, k, device="cuda")
            dzl = dZ[sh.dst_begin:sh.dst_end].contiguous()
            per.append(timed(lambda: (sh.spmm_fwd(va, ia, D, out=zl),
                                      sh.spmm_bwd(dzl, va, ia, D, out=gp))))
            pf.append(timed(lambda: sh.spmm_fwd(va, ia, D, out=zl)))
            pb.append(timed(lambda: sh.spmm_bwd(dzl, va, ia, D, out=gp)))
        r["world"][W] = {"rank_ms_max": max(per), "rank_ms_min": min(per),
                         "fwd_ms_max": max(pf), "bwd_ms_max": max(pb),
                         "tiles": shards[0].info()["tiles"], "tiles_T": shards[0].info()["tiles_T"],
                         "allgather_in_bytes": (W - 1) * m * k * 5,
                         "dense_allgather_in_bytes": (W - 1) * m * D * 4,
                         "reduce_scatter_bytes": (W - 1) * m * k * 4}
        del shards
    out["rels"][rel] = r
print(json.dumps(out))
