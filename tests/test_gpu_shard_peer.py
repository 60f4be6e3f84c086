"""f4, the exchange fused into the SpMM over peer memory (dr_shard_spmm_fwd_peer /
_bwd_peer / _inbox_reduce), with W virtual ranks on one GPU: every rank's kernels
read the other ranks' CBSR buffers and write the other ranks' inboxes in place
through a pointer table (on a multi-GPU node the same table holds NVLink-mapped
peer pointers, `peer_buffers`). The forward must equal the allgather path bit for
bit, the backward's per-source g the single-graph oracle within 1e-4."""
import numpy as np
import pytest

from gen import make_config
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")


@pytest.fixture(scope="module")
def designs():
    return {"C1": make_config("C1"), "C2s": make_config("C2", scale=0.1),
            "C4s": make_config("C4", scale=0.01)}


@pytest.mark.parametrize("name,D,k", [("C1", 16, 4), ("C2s", 64, 8), ("C4s", 128, 16)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("rel", ["near", "pins", "pinned"])
def test_shard_peer_exchange(designs, name, D, k, world, rel):
    d = designs[name]
    ptr, col, nd, ns = d.rel(rel)
    rng = np.random.default_rng(world * 13 + D)
    X = torch.as_tensor(rng.standard_normal((ns, D)).astype(np.float32)).cuda()
    dZ = torch.as_tensor(rng.standard_normal((nd, D)).astype(np.float32)).cuda()
    shards = [dr.Shard.from_design(d, rel, world, r) for r in range(world)]
    m = shards[0].max_src
    loc = []                                   # each rank's local CBSR buffer
    for sh in shards:
        xl = torch.zeros((m, D), device="cuda")
        xl[:sh.src_end - sh.src_begin] = X[sh.src_begin:sh.src_end]
        loc.append(dr.drelu_topk(xl, k))
    peers = [(v, i) for v, i in loc]
    # forward: in-place remote reads == the allgathered CBSR, bit for bit
    val_a = torch.cat([v for v, _ in loc])
    idx_a = torch.cat([i for _, i in loc])
    for sh in shards:
        z_peer = sh.spmm_fwd_peer(peers, D, k)
        z_ag = sh.spmm_fwd(val_a, idx_a, D)
        assert torch.equal(z_peer, z_ag)
    # backward: every rank writes its slot of every owner's inbox, owners sum
    inbox = [torch.full((world, m, k), float("nan"), device="cuda") for _ in range(world)]
    for sh in shards:
        sh.spmm_bwd_peer(dZ[sh.dst_begin:sh.dst_end].contiguous(), peers, D, k, inbox)
    g = []
    dxs = []
    for q, sh in enumerate(shards):
        g_l, dx_l = sh.inbox_reduce(inbox[q], loc[q][0], loc[q][1], D)
        g.append(g_l[:sh.src_end - sh.src_begin])
        dxs.append(dx_l[:sh.src_end - sh.src_begin])
    g = to_np(torch.cat(g))
    idx = torch.cat([loc[q][1][:sh.src_end - sh.src_begin] for q, sh in enumerate(shards)])
    c, s = O.normalisers(ptr, col, nd, ns, O.MEAN if rel != "pinned" else O.SYM)
    og = O.spmm_bwd(ptr, col, nd, ns, c, s, to_np(idx).astype(np.int32),
                    to_np(dZ).astype(np.float64))
    assert row_err(g, og) <= TOL
    dx = to_np(torch.cat(dxs))
    assert np.all(dx[O.densify(to_np(idx).astype(np.int32), np.ones_like(og), D) == 0] == 0)
    # determinism: a second pass gives the same bits
    for sh in shards:
        sh.spmm_bwd_peer(dZ[sh.dst_begin:sh.dst_end].contiguous(), peers, D, k, inbox)
    g2 = to_np(torch.cat([shards[q].inbox_reduce(inbox[q], loc[q][0], loc[q][1], D)[0]
                          [:shards[q].src_end - shards[q].src_begin] for q in range(world)]))
    assert np.array_equal(g, g2)
