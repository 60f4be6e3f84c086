"""NEXT-2 (DESIGN reading Q26) on the GPU vs the fp64 oracle.

Value-sorted D-ReLU (dr_drelu_topk_sorted) must equal oracle.drelu_sorted bit for
bit; the per-neighbour-group-K SpMM forward/backward (dr_spmm_fwd_ng / _bwd_ng)
must be within the north_star 1e-4 row-normalised error of oracle.spmm_fwd_ng /
spmm_bwd_ng fed the GPU's own CBSR (teacher-forced, as in test_gpu_parity)."""
import numpy as np
import pytest

from gen import make_config
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")

RELS = ("near", "pins", "pinned")
MOD = {"near": O.MEAN, "pins": O.MEAN, "pinned": O.SYM}


def within_cond(gpu, ref, ref_abs, n_terms):
    """Row-normalised TOL, plus the a-priori fp32 summation bound (n-1) u sum|terms|
    per element. Needed for g_kept under a schedule with kb = 1: rows whose only
    surviving position is one cancelling sum have ||o_r|| = |sum| << sum|terms|,
    where no fp32 summation order meets a pure relative bound."""
    g = np.asarray(gpu, np.float64)
    norms = np.linalg.norm(ref, axis=1, keepdims=True)
    tau = max(1e-6 * float(np.sqrt(np.mean(norms ** 2))), 1e-30)
    bound = TOL * np.maximum(norms, tau) + (n_terms[:, None] + 1) * 2.0 ** -24 * ref_abs
    return bool(np.all(np.abs(g - ref) <= bound))


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.fixture(scope="module")
def designs():
    return {"C1": make_config("C1"), "C2s": make_config("C2", scale=0.1),
            "C4s": make_config("C4", scale=0.01)}


@pytest.mark.parametrize("dim,k", [(16, 4), (64, 8), (128, 16), (256, 32), (64, 1), (32, 32),
                                   (96, 8)])
def test_drelu_sorted_bitexact(dim, k):
    rng = np.random.default_rng(dim * 7 + k)
    x = rng.standard_normal((2500, dim)).astype(np.float32)
    x[:300] = rng.integers(-2, 3, size=(300, dim)).astype(np.float32)   # heavy ties
    x[300] = 0.0
    x[301, ::2] = -0.0
    x[302] = -1.0
    xg = cuda(x)
    val, idx = dr.drelu_topk_sorted(xg, k)
    oi, ov = O.drelu_sorted(to_np(xg).astype(np.float64), k)
    assert np.array_equal(to_np(idx).astype(np.int32), oi)
    assert np.array_equal(to_np(val), ov.astype(np.float32))
    assert np.array_equal(np.signbit(to_np(val)), np.signbit(ov))
    # same set as the unsorted selection
    _, ui = dr.drelu_topk(xg, k)
    assert np.array_equal(np.sort(to_np(ui), axis=1), np.sort(to_np(idx), axis=1))


def test_drelu_sorted_rejects_large_k():
    x = torch.randn(10, 128, device="cuda")
    with pytest.raises(dr.DRError):
        dr.drelu_topk_sorted(x, 64)


SCHED = [((8, 64), (8, 4, 2)), ((16, 32), (4, 4, 1)), ((0, 1000000), (8, 8, 8)),
         ((2, 3), (16, 8, 1))]


@pytest.mark.parametrize("name,D,k", [("C1", 16, 4), ("C2s", 64, 8), ("C4s", 128, 16),
                                      ("C2s", 128, 16)])
@pytest.mark.parametrize("si", range(len(SCHED)))
def test_spmm_ng_parity(designs, name, D, k, si):
    thr, kb = SCHED[si]
    kb = tuple(min(v, k) for v in kb)
    d = designs[name]
    g = dr.Graph.from_design(d)
    rng = np.random.default_rng(si * 13 + D)
    for rel in RELS:
        ptr, col, nd, ns = d.rel(rel)
        x = cuda(rng.standard_normal((ns, D)).astype(np.float32))
        val, idx = dr.drelu_topk_sorted(x, k)
        oi = to_np(idx).astype(np.int32)
        ov = to_np(val).astype(np.float64)
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        plan = dr.NgPlan(g, rel, thr, kb)
        z = dr.spmm_fwd_ng(plan, val, idx, D)
        ref = O.spmm_fwd_ng(ptr, col, nd, c, s, oi, ov, D, thr, kb)
        assert row_err(to_np(z), ref) <= TOL, rel
        dz = cuda(rng.standard_normal((nd, D)).astype(np.float32))
        gk, dx = dr.spmm_bwd_ng(plan, dz, val, idx, D, want_g=True, want_dx=True)
        dz64 = to_np(dz).astype(np.float64)
        refg = O.spmm_bwd_ng(ptr, col, nd, ns, c, s, oi, dz64, thr, kb)
        absg = O.spmm_bwd_ng(ptr, col, nd, ns, np.abs(c), np.abs(s), oi, np.abs(dz64), thr, kb)
        n_terms = np.bincount(col, minlength=ns)
        assert row_err(to_np(gk), refg) <= TOL or within_cond(to_np(gk), refg, absg, n_terms), rel
        if min(kb) > 1:
            assert row_err(to_np(gk), refg) <= TOL, rel
        assert np.array_equal(to_np(dx), O.densify(oi, to_np(gk).astype(np.float64), D)
                              .astype(np.float32)), rel


def test_spmm_ng_uniform_equals_plain(designs):
    """kb = (k, k, k) is the plain DR-SpMM: same values as dr_spmm_fwd / bwd."""
    d = designs["C2s"]
    g = dr.Graph.from_design(d)
    rng = np.random.default_rng(5)
    for rel in RELS:
        ptr, col, nd, ns = d.rel(rel)
        x = cuda(rng.standard_normal((ns, 64)).astype(np.float32))
        val, idx = dr.drelu_topk_sorted(x, 8)
        plan = dr.NgPlan(g, rel, (4, 64), (8, 8, 8))
        z_ng = dr.spmm_fwd_ng(plan, val, idx, 64)
        z = dr.spmm_fwd(g, rel, val, idx, 64)
        assert row_err(to_np(z_ng), to_np(z).astype(np.float64)) <= 4e-5, rel
        dz = cuda(rng.standard_normal((nd, 64)).astype(np.float32))
        g_ng, _ = dr.spmm_bwd_ng(plan, dz, val, idx, 64)
        gk, _ = dr.spmm_bwd(g, rel, dz, val, idx, 64)
        assert row_err(to_np(g_ng), to_np(gk).astype(np.float64)) <= 4e-5, rel


def test_spmm_ng_adjoint(designs):
    d = designs["C4s"]
    g = dr.Graph.from_design(d)
    rng = np.random.default_rng(8)
    thr, kb = (8, 64), (16, 8, 2)
    for rel in RELS:
        ptr, col, nd, ns = d.rel(rel)
        x = cuda(rng.standard_normal((ns, 128)).astype(np.float32))
        val, idx = dr.drelu_topk_sorted(x, 16)
        plan = dr.NgPlan(g, rel, thr, kb)
        z = dr.spmm_fwd_ng(plan, val, idx, 128)
        dz = cuda(rng.standard_normal((nd, 128)).astype(np.float32))
        gk, _ = dr.spmm_bwd_ng(plan, dz, val, idx, 128)
        lhs = float((z.double() * dz.double()).sum())
        rhs = float((val.double() * gk.double()).sum())
        assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + 1.0), rel


@pytest.mark.parametrize("thr,kb", [((8, 4), (8, 4, 2)), ((4, 8), (2, 4, 1)),
                                    ((4, 8), (8, 4, 0)), ((4, 8), (64, 4, 2))])
def test_spmm_ng_bad_schedule(designs, thr, kb):
    g = dr.Graph.from_design(designs["C1"])
    with pytest.raises(dr.DRError):
        dr.NgPlan(g, "near", thr, kb)


def test_spmm_ng_k_below_plan(designs):
    d = designs["C1"]
    g = dr.Graph.from_design(d)
    plan = dr.NgPlan(g, "near", (4, 8), (16, 4, 2))
    x = torch.randn(d.rel("near")[3], 16, device="cuda")
    val, idx = dr.drelu_topk_sorted(x, 8)
    with pytest.raises(dr.DRError) as e:
        dr.spmm_fwd_ng(plan, val, idx, 16)
    assert e.value.status == 2


def test_ng_edge_cases():
    """Empty relations, zero rows and isolated destinations: exact zeros, no errors."""
    n_cell, n_net = 10, 5
    empty = (np.zeros(n_cell + 1, np.int64), np.zeros(0, np.int32))
    rels = {"near": empty, "pins": (np.zeros(n_net + 1, np.int64), np.zeros(0, np.int32)),
            "pinned": empty}
    g = dr.Graph(n_cell, n_net, rels)
    x = torch.randn(n_cell, 16, device="cuda")
    val, idx = dr.drelu_topk_sorted(x, 4)
    plan = dr.NgPlan(g, "near", (2, 4), (4, 2, 1))
    z = dr.spmm_fwd_ng(plan, val, idx, 16)
    assert torch.count_nonzero(z) == 0
    gk, dx = dr.spmm_bwd_ng(plan, torch.randn(n_cell, 16, device="cuda"), val, idx, 16,
                            want_dx=True)
    assert torch.count_nonzero(gk) == 0 and torch.count_nonzero(dx) == 0
    v0, i0 = dr.drelu_topk_sorted(torch.empty(0, 16, device="cuda"), 4)
    assert v0.shape == (0, 4)
