"""Tensor-core tiled SpMM (csrc/tspmm.cu) against the fp64 oracle and against the
SIMT kernels (dr.debug_set("tspmm", 0)), on the near relation (the only one tiled: unit
weights, mean degree >= 8). Covers symmetric and asymmetric near (separate CSC
tiles), isolated rows (empty-halo tiles), every supported (D, k), the
standalone ABI backward (dZ row scale applied in the converters) and determinism."""
import numpy as np
import pytest

from gen import make_config
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.fixture(scope="module")
def designs():
    return {"C2s": make_config("C2", scale=0.1), "C4s": make_config("C4", scale=0.01)}


def _asym_near(d, drop=0.1, isolate=50, seed=3):
    """near with a random `drop` share of edges removed (no longer symmetric) and
    the first `isolate` cells' rows emptied (isolated destinations)."""
    ptr, col = d.rel("near")[:2]
    rng = np.random.default_rng(seed)
    keep = rng.random(col.size) >= drop
    rows = np.repeat(np.arange(d.n_cell), np.diff(ptr))
    keep &= rows >= isolate
    col2 = col[keep]
    cnt = np.bincount(rows[keep], minlength=d.n_cell)
    ptr2 = np.zeros(d.n_cell + 1, np.int64)
    ptr2[1:] = np.cumsum(cnt)
    return ptr2, col2.astype(np.int32)


def _fwd_bwd(g, D, k, seed, n_src, n_dst):
    rng = np.random.default_rng(seed)
    x = cuda(rng.standard_normal((n_src, D)).astype(np.float32))
    val, idx = dr.drelu_topk(x, k)
    z = dr.spmm_fwd(g, "near", val, idx, D)
    dz = cuda(rng.standard_normal((n_dst, D)).astype(np.float32))
    gk, dx = dr.spmm_bwd(g, "near", dz, val, idx, D, want_g=True, want_dx=True)
    return val, idx, dz, z, gk, dx


def test_tiles_built(designs):
    d = designs["C2s"]
    info = dr.Graph.from_design(d).info()
    assert info["tiles"][0] > 0 and info["tiles_T"][0] == info["tiles"][0]     # symmetric: shared
    assert info["chunks"][0] >= info["tiles"][0]
    assert info["tiles"][1] == 0 and info["tiles"][2] == 0                      # pins/pinned: SIMT
    assert dr.Graph.from_design(d, flags=2).info()["tiles"][0] == 0              # identity order
    ptr, col = _asym_near(d)
    rels = {r: d.rel(r)[:2] for r in ("pins", "pinned")}
    rels["near"] = (ptr, col)
    ia = dr.Graph(d.n_cell, d.n_net, rels).info()
    assert ia["tiles"][0] > 0 and ia["tiles_T"][0] > 0


@pytest.mark.parametrize("name,D,k", [("C2s", 64, 8), ("C4s", 128, 16), ("C2s", 128, 4),
                                      ("C2s", 64, 32), ("C4s", 64, 16), ("C2s", 128, 32)])
def test_tspmm_matches_oracle_and_simt(designs, name, D, k, knob):
    d = designs[name]
    g = dr.Graph.from_design(d)
    assert g.info()["tiles"][0] > 0
    ptr, col, nd, ns = d.rel("near")
    val, idx, dz, z, gk, dx = _fwd_bwd(g, D, k, 5, ns, nd)
    c, s = O.normalisers(ptr, col, nd, ns, O.MEAN)
    oi = to_np(idx).astype(np.int32)
    ref_z = O.spmm_fwd(ptr, col, nd, c, s, oi, to_np(val).astype(np.float64), D)
    assert row_err(to_np(z), ref_z) <= TOL
    ref_g = O.spmm_bwd(ptr, col, nd, ns, c, s, oi, to_np(dz).astype(np.float64))
    assert row_err(to_np(gk), ref_g) <= TOL
    assert np.array_equal(to_np(dx), O.densify(oi, to_np(gk).astype(np.float64), D).astype(np.float32))
    # same results as the SIMT kernels up to fp32 rounding
    knob("tspmm", 0, 1)
    z_s = dr.spmm_fwd(g, "near", val, idx, D)
    gk_s, _ = dr.spmm_bwd(g, "near", dz, val, idx, D)
    # (bf16 hi/lo split: |x - hi - lo| <= 2^-17 |x| per term on the tensor-core side)
    assert row_err(to_np(z), to_np(z_s).astype(np.float64)) <= 4e-5
    assert row_err(to_np(gk), to_np(gk_s).astype(np.float64)) <= 4e-5


@pytest.mark.parametrize("D,k", [(64, 8), (128, 16)])
def test_tspmm_asymmetric_and_isolated(designs, D, k):
    d = designs["C2s"] if D == 64 else designs["C4s"]
    ptr, col = _asym_near(d)
    rels = {r: d.rel(r)[:2] for r in ("pins", "pinned")}
    rels["near"] = (ptr, col)
    g = dr.Graph(d.n_cell, d.n_net, rels)
    info = g.info()
    assert info["tiles"][0] > 0 and info["tiles_T"][0] > 0
    n = d.n_cell
    val, idx, dz, z, gk, dx = _fwd_bwd(g, D, k, 9, n, n)
    c, s = O.normalisers(ptr, col, n, n, O.MEAN)
    oi = to_np(idx).astype(np.int32)
    ref_z = O.spmm_fwd(ptr, col, n, c, s, oi, to_np(val).astype(np.float64), D)
    assert row_err(to_np(z), ref_z) <= TOL
    assert np.all(to_np(z)[:50] == 0.0)                          # isolated destinations
    ref_g = O.spmm_bwd(ptr, col, n, n, c, s, oi, to_np(dz).astype(np.float64))
    assert row_err(to_np(gk), ref_g) <= TOL


def test_tspmm_deterministic(designs):
    d = designs["C4s"]
    g = dr.Graph.from_design(d)
    a = _fwd_bwd(g, 128, 16, 1, d.n_cell, d.n_cell)
    b = _fwd_bwd(g, 128, 16, 1, d.n_cell, d.n_cell)
    for x, y in zip(a[3:], b[3:]):
        assert torch.equal(x, y)
