"""f4: a HeteroConv layer sharded by destination rows (dr_shard_layer_*), every
exchange through peer memory, with W virtual ranks on one GPU (pointer tables
of local buffers; on a node: NVLink-mapped peers). The ranks' outputs,
concatenated, and their weight-gradient contributions, summed, must match the
single-graph fp64 oracle layer (Eq. 2-14) within 1e-4 row-normalised, on an
instance without merge near-ties (every margin >= 1e-5 of its row, so the fp32
and fp64 sides take the same decisions)."""
import numpy as np
import pytest

from gen import make_config, make_params
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")

D, K = 32, 8


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.fixture(scope="module")
def instance():
    d = make_config("C2", scale=0.02, D=D)
    G = O.OGraph(d)
    P = make_params(D, D, D, 1, seed=4)
    W = O.layer_params(P, 0)
    for seed in range(200):
        rng = np.random.default_rng(seed)
        xc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
        xn = rng.standard_normal((d.n_net, D)).astype(np.float32)
        # D-ReLU of the fp32 inputs is exact on both sides; the merge decisions are
        # taken on fp32 (GPU) vs fp64 (oracle) Y: keep every margin >= 1e-5 of the row
        yc, yn, tape = O.layer_fwd(G, W, xc, xn, K, K)
        marg = np.abs(tape["y_near"] - tape["y_pinned"])
        nrm = np.linalg.norm(np.maximum(tape["y_near"], tape["y_pinned"]), axis=1, keepdims=True)
        ok = bool(np.all(marg >= 1e-5 * nrm))
        if ok:
            dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
            dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
            return d, G, P, W, xc, xn, yc, yn, tape, dyc, dyn
    pytest.skip("no tie-free instance")


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_layer_matches_oracle(instance, world):
    d, G, P, W, xc, xn, oyc, oyn, otape, dyc, dyn = instance
    # one cell and one net partition for all three relations
    cp, _ = dr.shard_plan(*d.rel("near")[:2], d.rel("near")[3], world)
    npart, _ = dr.shard_plan(*d.rel("pins")[:2], d.rel("pins")[3], world)
    layers, shards = [], []
    for r in range(world):
        sn = dr.Shard.from_design(d, "near", world, r, dst_part=cp, src_part=cp)
        sp = dr.Shard.from_design(d, "pins", world, r, dst_part=npart, src_part=cp)
        sq = dr.Shard.from_design(d, "pinned", world, r, dst_part=cp, src_part=npart)
        shards.append((sn, sp, sq))
        layers.append(dr.ShardLayer(sn, sp, sq))
    mc, mn = layers[0].m_cell, layers[0].m_net
    Wt = {kk.split(".", 1)[1]: cuda(v) for kk, v in P.items() if kk.startswith("l0.")}
    L = dr.Layer(Wt, D, D, D, K, K)
    # step 1: every rank's local CBSR (its rows, zero-padded to max_src)
    pc, pn = [], []
    for r in range(world):
        c0, c1 = int(cp[r]), int(cp[r + 1])
        n0, n1 = int(npart[r]), int(npart[r + 1])
        xl = torch.zeros((mc, D), device="cuda")
        xl[:c1 - c0] = cuda(xc[c0:c1])
        pc.append(dr.drelu_topk(xl, K))
        xl = torch.zeros((mn, D), device="cuda")
        xl[:n1 - n0] = cuda(xn[n0:n1])
        pn.append(dr.drelu_topk(xl, K))
    # step 2: forward
    outs = [sl.fwd(L, pc, pn) for sl in layers]
    yc = np.concatenate([to_np(o[0]) for o in outs])
    yn = np.concatenate([to_np(o[1]) for o in outs])
    assert row_err(yc, oyc) <= TOL
    assert row_err(yn, oyn) <= TOL
    # step 3: backward into the owners' inboxes; weight gradients summed over ranks
    inbox_c = [torch.full((2, world, mc, K), float("nan"), device="cuda") for _ in range(world)]
    inbox_n = [torch.full((world, mn, K), float("nan"), device="cuda") for _ in range(world)]
    gsum = None
    for r, sl in enumerate(layers):
        c0, c1 = int(cp[r]), int(cp[r + 1])
        n0, n1 = int(npart[r]), int(npart[r + 1])
        gr = sl.bwd(L, outs[r][2], cuda(dyc[c0:c1]), cuda(dyn[n0:n1]), pc, pn, inbox_c, inbox_n)
        gsum = {kk: to_np(v).astype(np.float64) for kk, v in gr.items()} if gsum is None else \
            {kk: gsum[kk] + to_np(v) for kk, v in gr.items()}
    # step 4: every owner's dX
    dx = [sl.dx(L, outs[r][2], pc, pn, inbox_c[r], inbox_n[r]) for r, sl in enumerate(layers)]
    dxc = np.concatenate([to_np(a) for a, _ in dx])
    dxn = np.concatenate([to_np(b) for _, b in dx])
    og, odxc, odxn = O.layer_bwd(G, W, otape, dyc, dyn, need_dx=True)
    for kk in og:
        assert row_err(gsum[kk], og[kk]) <= TOL, kk
    assert row_err(dxc, odxc) <= TOL
    assert row_err(dxn, odxn) <= TOL
    assert np.all(dxc[odxc == 0] == 0)
