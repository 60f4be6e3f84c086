"""World-size-2 data-parallel host logic on CPU (gloo): NCCL-id style byte
broadcast, max-over-ranks timing, equal-nnz batch packing, and the DP gradient
semantics dr_train_step implements (allreduce SUM of per-rank gradients, then
1/W in Adam) == the oracle's mean of rank gradients == the gradient of the
union batch when per-rank batches have equal cell counts."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import disjoint_union, make_design, make_params
from oracle import oracle as O
from paper_2508_16769_b200 import dist as ddp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _designs():
    return [make_design(f"g{i}", 40, 300 + i, d_cell=16, d_net=16, near_mean=5, near_cap=16,
                        pins_mean=2.5, pins_dmax=10, n_net=20) for i in range(4)]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = ddp.broadcast_bytes(bytes(range(128)) if rank == 0 else None)
        assert uid == bytes(range(128))
        assert ddp.max_over_ranks(10.0 * (rank + 1)) == 10.0 * world
        designs = _designs()
        batches = ddp.pack_batches([d.near_col.size for d in designs], world)
        mine = disjoint_union([designs[i] for i in batches[rank]])
        P = make_params(16, 16, 16, 2, seed=3)
        _, g, _ = O.model_fwd_bwd(O.OGraph(mine), P, 2, 4, 4, mine.x_cell, mine.x_net,
                                  mine.labels)
        keys = sorted(g)
        flat = torch.tensor(np.concatenate([g[k].reshape(-1) for k in keys]))
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)          # what ncclAllReduce does
        flat /= world                                        # the 1/W folded into Adam
        out[rank] = flat.numpy().copy()
    finally:
        dist.destroy_process_group()


def test_dp_two_ranks_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert np.array_equal(out[0], out[1])                    # every rank holds the same mean
    designs = _designs()
    batches = ddp.pack_batches([d.near_col.size for d in designs], world)
    P = make_params(16, 16, 16, 2, seed=3)
    per_rank = []
    for b in batches:
        u = disjoint_union([designs[i] for i in b])
        per_rank.append(O.model_fwd_bwd(O.OGraph(u), P, 2, 4, 4, u.x_cell, u.x_net, u.labels)[1])
    mean = O.dp_mean(per_rank)
    keys = sorted(mean)
    ref = np.concatenate([mean[k].reshape(-1) for k in keys])
    assert np.allclose(out[0], ref, rtol=1e-12, atol=1e-15)
    # equal cell counts per rank => the DP mean is the gradient of the union batch
    u = disjoint_union(designs)
    gu = O.model_fwd_bwd(O.OGraph(u), P, 2, 4, 4, u.x_cell, u.x_net, u.labels)[1]
    assert np.allclose(ref, np.concatenate([gu[k].reshape(-1) for k in keys]), rtol=1e-10,
                       atol=1e-13)


def test_pack_batches_balances_and_covers():
    rng = np.random.default_rng(0)
    work = rng.integers(280_000, 530_000, size=250)          # Table 1 range of edges per graph
    for world in (1, 2, 4, 8):
        b = ddp.pack_batches(work, world)
        assert sorted(i for x in b for i in x) == list(range(250))
        assert ddp.imbalance(work, b) < 1.02
    assert ddp.pack_batches([5, 1, 1, 1, 1, 1], 2) == [[0], [1, 2, 3, 4, 5]]
