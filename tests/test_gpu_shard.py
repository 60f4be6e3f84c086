"""Single-graph multi-GPU DR-SpMM through the C ABI on one GPU.

W virtual ranks in one process: every rank's dr_shard is created, the exchanges
are assembled test-side (the allgather is a concatenation of the padded rank
blocks, the reduce-scatter a sum + slice), and the ranks' dr_shard_spmm_fwd /
_bwd outputs must reproduce the single-graph oracle within the north_star 1e-4
row-normalised error. World 1 runs the real NCCL collectives (a one-rank
communicator); the multi-rank NCCL path needs several GPUs and is covered on
CPU by tests/test_shard_gloo.py."""
import numpy as np
import pytest

from gen import make_config
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")

MOD = {"near": O.MEAN, "pins": O.MEAN, "pinned": O.SYM}


@pytest.fixture(scope="module")
def designs():
    return {"C1": make_config("C1"), "C2s": make_config("C2", scale=0.1),
            "C4s": make_config("C4", scale=0.01)}


def _virtual(d, rel, world, D, k, seed):
    ptr, col, nd, ns = d.rel(rel)
    rng = np.random.default_rng(seed)
    X = torch.as_tensor(rng.standard_normal((ns, D)).astype(np.float32)).cuda()
    dZ = torch.as_tensor(rng.standard_normal((nd, D)).astype(np.float32)).cuda()
    shards = [dr.Shard.from_design(d, rel, world, r) for r in range(world)]
    m = shards[0].max_src
    loc = []
    for sh in shards:
        xl = torch.zeros((m, D), device="cuda")
        xl[:sh.src_end - sh.src_begin] = X[sh.src_begin:sh.src_end]
        loc.append(dr.drelu_topk(xl, k))
    val_a = torch.cat([v for v, _ in loc])
    idx_a = torch.cat([i for _, i in loc])
    z = torch.cat([sh.spmm_fwd(val_a, idx_a, D) for sh in shards])
    g_sum = sum(sh.spmm_bwd(dZ[sh.dst_begin:sh.dst_end].contiguous(), val_a, idx_a, D)
                for sh in shards)
    g = torch.cat([g_sum[q * m: q * m + sh.src_end - sh.src_begin]
                   for q, sh in enumerate(shards)])
    # the global CBSR those ranks hold, in source order
    idx = torch.cat([loc[q][1][:sh.src_end - sh.src_begin] for q, sh in enumerate(shards)])
    val = torch.cat([loc[q][0][:sh.src_end - sh.src_begin] for q, sh in enumerate(shards)])
    return ptr, col, nd, ns, z, g, val, idx, dZ, shards


@pytest.mark.parametrize("name,D,k", [("C1", 16, 4), ("C2s", 64, 8), ("C4s", 128, 16)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_virtual_ranks_parity(designs, name, D, k, world):
    d = designs[name]
    for rel in ("near", "pins", "pinned"):
        ptr, col, nd, ns, z, g, val, idx, dZ, _ = _virtual(d, rel, world, D, k, world * 31 + D)
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        oi, ov = to_np(idx).astype(np.int32), to_np(val).astype(np.float64)
        assert row_err(to_np(z), O.spmm_fwd(ptr, col, nd, c, s, oi, ov, D)) <= TOL, rel
        ref = O.spmm_bwd(ptr, col, nd, ns, c, s, oi, to_np(dZ).astype(np.float64))
        assert row_err(to_np(g), ref) <= TOL, rel


def test_shard_near_blocks_tiled_optin(knob):
    """DR_SHARD_TILES=1 (opt-in): with node ids in a locality order, near's blocks
    (unit weights, dense neighbourhoods) run the tensor-core tiled forward, with
    the same parity; the SSpMM stays SIMT unless DR_SHARD_TILES_T=1."""
    knob("shard_tiles", 1, 0)
    d = make_config("C2", scale=0.1, order="spatial")
    for world in (1, 2, 4):
        for q in range(world):
            i = dr.Shard.from_design(d, "near", world, q).info()
            assert i["tiles"] > 0, (world, q)
        ptr, col, nd, ns, z, g, val, idx, dZ, _ = _virtual(d, "near", world, 64, 8, world)
        c, s = O.normalisers(ptr, col, nd, ns, MOD["near"])
        oi, ov = to_np(idx).astype(np.int32), to_np(val).astype(np.float64)
        assert row_err(to_np(z), O.spmm_fwd(ptr, col, nd, c, s, oi, ov, 64)) <= TOL


def test_shard_world1_equals_single_graph(designs):
    """One rank: bit-identical to dr_spmm_fwd / dr_spmm_bwd on the SIMT path."""
    d = designs["C2s"]
    g = dr.Graph.from_design(d, flags=0)
    for rel in ("pins", "pinned"):           # (near runs the tiled kernel on a full graph)
        ptr, col, nd, ns, z, gk, val, idx, dZ, _ = _virtual(d, rel, 1, 64, 8, 5)
        assert row_err(to_np(z), to_np(dr.spmm_fwd(g, rel, val, idx, 64)).astype(np.float64)) <= 1e-6
        g2, _ = dr.spmm_bwd(g, rel, dZ, val, idx, 64)
        assert row_err(to_np(gk), to_np(g2).astype(np.float64)) <= 1e-6


def test_shard_nccl_world1(designs):
    d = designs["C2s"]
    comm = dr.nccl_comm_init(dr.nccl_unique_id(), 1, 0)
    try:
        sh = dr.Shard.from_design(d, "near", 1, 0)
        x = torch.randn(d.n_cell, 64, device="cuda")
        vl, il = dr.drelu_topk(x, 8)
        va, ia = sh.allgather_cbsr(vl, il, 64, comm=comm)
        assert torch.equal(va, vl) and torch.equal(ia, il)
        dz = torch.randn(d.n_cell, 64, device="cuda")
        gp = sh.spmm_bwd(dz, va, ia, 64)
        gl, dx = sh.reduce_scatter_g(gp, vl, il, 64, want_dx=True, comm=comm)
        torch.cuda.synchronize()
        assert torch.equal(gl, gp)
        ref = O.densify(to_np(il).astype(np.int32), to_np(gl).astype(np.float64), 64)
        assert np.array_equal(to_np(dx), ref.astype(np.float32))
        sh2 = dr.Shard.from_design(d, "near", 2, 0)
        with pytest.raises(dr.DRError):           # communicator of 1 rank for a 2-rank shard
            sh2.allgather_cbsr(torch.zeros(sh2.max_src, 8, device="cuda"),
                               torch.zeros(sh2.max_src, 8, device="cuda", dtype=torch.uint8),
                               64, comm=comm)
    finally:
        dr.nccl_comm_destroy(comm)


def test_shard_bad_partition(designs):
    d = designs["C1"]
    ptr, col, nd, ns = d.rel("near")
    with pytest.raises(dr.DRError):
        dr.Shard(ptr, col, ns, 2, 0, dst_part=[0, nd + 1, nd])
    with pytest.raises(dr.DRError):
        dr.Shard(ptr, col, ns, 2, 2)


def test_shard_more_ranks_than_rows():
    """world larger than the row count: empty ranks own no rows; the union is still exact."""
    d = make_config("C1")                        # 64 cells, 32 nets
    for rel in ("pins", "pinned"):
        ptr, col, nd, ns, z, g, val, idx, dZ, shards = _virtual(d, rel, 48, 16, 4, 3)
        assert any(sh.dst_end == sh.dst_begin for sh in shards)
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        oi, ov = to_np(idx).astype(np.int32), to_np(val).astype(np.float64)
        assert row_err(to_np(z), O.spmm_fwd(ptr, col, nd, c, s, oi, ov, 16)) <= TOL
        ref = O.spmm_bwd(ptr, col, nd, ns, c, s, oi, to_np(dZ).astype(np.float64))
        assert row_err(to_np(g), ref) <= TOL


def test_shard_empty_relation():
    ptr, col = np.zeros(11, np.int64), np.zeros(0, np.int32)
    for world in (1, 2):
        shards = [dr.Shard(ptr, col, 7, world, q) for q in range(world)]
        m = shards[0].max_src
        va = torch.randn(world * m, 4, device="cuda")
        ia = torch.zeros(world * m, 4, device="cuda", dtype=torch.uint8)
        ia[:] = torch.arange(4, dtype=torch.uint8, device="cuda")
        for sh in shards:
            z = sh.spmm_fwd(va, ia, 16)
            assert z.shape[0] == sh.dst_end - sh.dst_begin and torch.count_nonzero(z) == 0
            gp = sh.spmm_bwd(torch.randn(sh.dst_end - sh.dst_begin, 16, device="cuda"), va, ia, 16)
            assert torch.count_nonzero(gp) == 0
