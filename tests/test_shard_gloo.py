"""Single-graph multi-GPU protocol on CPU, world size 2 (gloo):
the 1-D destination partition of dr_shard_plan (libdr host code), local D-ReLU
of each rank's sources, allgather of the compact CBSR into the padded source
space, the row-block SpMM with GLOBAL normalisers, and the reduce-scatter of the
per-source partial g. The union of the ranks' Z rows and their reduced g must
equal the single-graph oracle (fp64, summation order only)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import make_config
from oracle import oracle as O
import paper_2508_16769_b200 as dr

D, K = 16, 4
MOD = {"near": O.MEAN, "pins": O.MEAN, "pinned": O.SYM}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(rel):
    d = make_config("C1")
    ptr, col, nd, ns = d.rel(rel)
    rng = np.random.default_rng(7)
    return d, ptr, col, nd, ns, rng.standard_normal((ns, D)), rng.standard_normal((nd, D))


def _worker(rank, world, port, rel, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, ptr, col, nd, ns, X, dZ = _inputs(rel)
        dp, sp = dr.shard_plan(ptr, col, ns, world, dr.DEFAULT_MODULES[rel])
        m = int(np.max(np.diff(sp)))
        # this rank's sources: D-ReLU, padded to m rows (padding: zero values)
        idx_l = np.zeros((m, K), np.int32)
        val_l = np.zeros((m, K))
        n_own = sp[rank + 1] - sp[rank]
        if n_own:
            idx_l[:n_own], val_l[:n_own] = O.drelu(X[sp[rank]:sp[rank + 1]], K)
        idx_t = [torch.zeros((m, K), dtype=torch.int32) for _ in range(world)]
        val_t = [torch.zeros((m, K), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(idx_t, torch.from_numpy(idx_l))
        dist.all_gather(val_t, torch.from_numpy(val_l))
        idx_a, val_a = torch.cat(idx_t).numpy(), torch.cat(val_t).numpy()
        # padded source ids and the global normalisers
        owner = np.searchsorted(sp, np.arange(ns), side="right") - 1
        pad = owner * m + (np.arange(ns) - sp[owner])
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        s_pad = np.ones(world * m)
        s_pad[pad] = s
        r0, r1 = dp[rank], dp[rank + 1]
        lptr = ptr[r0:r1 + 1] - ptr[r0]
        lcol = pad[col[ptr[r0]:ptr[r1]]].astype(np.int32)
        z_l = O.spmm_fwd(lptr, lcol, r1 - r0, c[r0:r1], s_pad, idx_a, val_a, D)
        g_part = O.spmm_bwd(lptr, lcol, r1 - r0, world * m, c[r0:r1], s_pad, idx_a, dZ[r0:r1])
        gt = torch.from_numpy(g_part)
        dist.all_reduce(gt)                   # reduce-scatter == allreduce + own block
        g_l = gt.numpy()[rank * m: rank * m + n_own]
        out[rank] = (z_l, g_l, int(r0), int(r1), int(sp[rank]), int(sp[rank + 1]))
    finally:
        dist.destroy_process_group()


def _check(rel):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), rel, out), nprocs=world, join=True)
    d, ptr, col, nd, ns, X, dZ = _inputs(rel)
    idx, val = O.drelu(X, K)
    c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
    z = O.spmm_fwd(ptr, col, nd, c, s, idx, val, D)
    g = O.spmm_bwd(ptr, col, nd, ns, c, s, idx, dZ)
    zs, gs = np.zeros_like(z), np.zeros_like(g)
    for r in range(world):
        z_l, g_l, r0, r1, s0, s1 = out[r]
        zs[r0:r1] = z_l
        gs[s0:s1] = g_l
    assert np.allclose(zs, z, rtol=1e-12, atol=1e-14)
    assert np.allclose(gs, g, rtol=1e-12, atol=1e-14)


def test_shard_protocol_near_gloo():
    _check("near")


def test_shard_protocol_pinned_gloo():
    _check("pinned")


def test_shard_plan_balance():
    d = make_config("C2", scale=0.1)
    for rel in ("near", "pins", "pinned"):
        ptr, col, nd, ns = d.rel(rel)
        maxdeg = int(np.diff(ptr).max())
        for world in (1, 2, 3, 8):
            dp, sp = dr.shard_plan(ptr, col, ns, world, dr.DEFAULT_MODULES[rel])
            assert dp[0] == 0 and dp[-1] == nd and np.all(np.diff(dp) >= 0)
            assert sp[0] == 0 and sp[-1] == ns and np.all(np.diff(sp) >= 0)
            per = np.diff(ptr[dp])
            assert per.max() <= ptr[-1] / world + maxdeg + 1
            if nd == ns:
                assert np.array_equal(dp, sp)
