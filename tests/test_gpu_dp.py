"""Data-parallel training path of libdr on one GPU (north_star:
"a single NCCL gradient allreduce over NVLink per step").

* A trainer given a world-1 NCCL communicator runs the in-library
  ncclAllReduce of the flat gradient (also inside the captured CUDA graph of
  the step) and must be bit-identical to the trainer without one.
* The trainer's CUDA-graph cache is LRU-bounded: stepping over more distinct
  input buffers than it holds must keep producing the same parameters as a
  trainer stepping on one set of buffers.
* The packed C5 batches of a data-parallel step (disjoint union of designs,
  reading Q24) give the oracle's gradient of the union."""
import numpy as np
import pytest

from gen import make_design, make_params
from gen.circuit import disjoint_union
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
dr = pytest.importorskip("paper_2508_16769_b200")


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def _small(seed=3, n=600, D=32):
    d = make_design("dp", n, seed, d_cell=D, d_net=D, near_mean=12.0, near_cap=64,
                    pins_mean=2.8, pins_dmax=40)
    return d, make_params(D, D, D, 2, seed=seed)


def test_trainer_nccl_world1_bit_identical():
    D, k = 32, 8
    d, P = _small()
    g = dr.Graph.from_design(d)
    xc, xn, y = cuda(d.x_cell), cuda(d.x_net), cuda(d.labels)
    comm = dr.nccl_comm_init(dr.nccl_unique_id(), 1, 0)
    try:
        fa = cuda(dr.flatten_params(P, 2))
        fb = fa.clone()
        ta = dr.Trainer(fa, 2, D, D, D, k, k)
        tb = dr.Trainer(fb, 2, D, D, D, k, k, nccl_comm=comm)
        ga, gb = torch.empty_like(fa), torch.empty_like(fb)
        la = ta.step(g, xc, xn, y, grad_out=ga)
        lb = tb.step(g, xc, xn, y, grad_out=gb)
        assert la == lb and torch.equal(ga, gb)
        for _ in range(6):               # eager, captured (allreduce in the graph), replays
            la, lb = ta.step(g, xc, xn, y), tb.step(g, xc, xn, y)
            assert la == lb
        torch.cuda.synchronize()
        assert torch.equal(fa, fb)
        ta.close()
        tb.close()
    finally:
        dr.nccl_comm_destroy(comm)


def test_graph_cache_eviction_keeps_results():
    """> 128 distinct (graph, buffers) keys: the cache evicts and re-captures
    without changing the trajectory."""
    D, k = 32, 8
    d, P = _small(seed=4, n=300)
    g = dr.Graph.from_design(d)
    fa = cuda(dr.flatten_params(P, 2))
    fb = fa.clone()
    ta = dr.Trainer(fa, 2, D, D, D, k, k, lr=1e-3)
    tb = dr.Trainer(fb, 2, D, D, D, k, k, lr=1e-3)
    fixed = (cuda(d.x_cell), cuda(d.x_net), cuda(d.labels))
    pool = [tuple(t.clone() for t in fixed) for _ in range(150)]
    for step in range(3 * 150 + 30):
        la = ta.step(g, *fixed)
        # each buffer set 3 steps in a row (eager, capture, replay), 150 sets in turn
        lb = tb.step(g, *pool[(step // 3) % 150])
        assert la == lb, step
    torch.cuda.synchronize()
    assert torch.equal(fa, fb)


def test_packed_batch_gradient_is_union_oracle():
    """A rank's packed batch = disjoint union of designs (Q24): the GPU step's
    gradient equals the oracle gradient of the union (tie-free instance)."""
    D, k = 16, 4
    for base in range(40, 200):
        parts = [make_design(f"p{q}", 80 + 10 * q, base * 10 + q, d_cell=D, d_net=D,
                             near_mean=6.0, near_cap=16, pins_mean=2.5, pins_dmax=12)
                 for q in range(3)]
        u = disjoint_union(parts)
        P = make_params(D, D, D, 2, seed=base)
        G = O.OGraph(u)
        ok, hc, hn = True, u.x_cell, u.x_net
        for l in range(2):
            for X in (hc, hn):
                s = -np.sort(-np.asarray(X, np.float64), axis=1)
                ok &= bool(np.all(s[:, k - 1] - s[:, k] >= 1e-4))
            hc, hn, tape = O.layer_fwd(G, O.layer_params(P, l), hc, hn, k, k)
            ok &= bool(np.abs(tape["y_near"] - tape["y_pinned"]).min() >= 1e-4)
        if ok:
            break
    assert ok
    g = dr.Graph.from_design(u)
    flat = cuda(dr.flatten_params(P, 2))
    tr = dr.Trainer(flat, 2, D, D, D, k, k)
    grad = torch.empty_like(flat)
    loss = tr.step(g, cuda(u.x_cell), cuda(u.x_net), cuda(u.labels), grad_out=grad)
    oloss, og, _ = O.model_fwd_bwd(G, P, 2, k, k, u.x_cell, u.x_net, u.labels)
    assert abs(loss - oloss) <= TOL * abs(oloss)
    ref = dr.flatten_params(og, 2).astype(np.float64)
    assert row_err(to_np(grad)[None, :], ref[None, :]) <= TOL
