"""Full-size GPU parity of the §8 f2-f4 rows (BASELINE configs[1] C2 and
configs[3] C4), the same bars as tests/test_gpu_fullsize.py:

* f2 NEXT-2 at C4: value-sorted D-ReLU bit-exact on sampled rows (random, the
  heaviest, every hub); the per-neighbour-group-K SpMM forward on sampled
  destination rows and the backward g on sampled source rows, each computed by
  the oracle definition row by row from the GPU's CBSR;
* f3 per-edge-type k at C2: one layer with k_pins = 4 (k_cell = k_net = 8),
  every row, teacher-forced against oracle.layer_fwd / layer_bwd(k_p);
* f4 sharding at C4: 8 virtual ranks per relation; the union of the ranks'
  Z rows and the reduced g equal the single-graph GPU results (tensor-core
  tiled for near) and the oracle on sampled rows."""
import numpy as np
import pytest

from gen import make_config, make_params
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
dr = pytest.importorskip("paper_2508_16769_b200")

MOD = {"near": O.MEAN, "pins": O.MEAN, "pinned": O.SYM}
TRANSPOSE = {"near": "near", "pins": "pinned", "pinned": "pins"}


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.fixture(scope="module")
def c4():
    return make_config("C4")


def _sample(n, deg, rng, extra=()):
    heavy = np.argsort(-deg, kind="stable")[:64]
    rnd = rng.choice(n, size=min(n, 2000), replace=False)
    return np.unique(np.concatenate([heavy, rnd, np.asarray(extra, np.int64)])).astype(np.int64)


def _fwd_rows(ptr, col, rows, c, s, idx, val, D, K=None):
    """Eq. 5 for the given destination rows; K[i] (optional) = prefix length."""
    out = np.zeros((rows.size, D))
    for r, i in enumerate(rows):
        nb = col[ptr[i]:ptr[i + 1]]
        kk = idx.shape[1] if K is None else int(K[i])
        for t in range(kk):
            np.add.at(out[r], idx[nb, t], s[nb] * val[nb, t])
    return c[rows][:, None] * out


def _bwd_rows(tptr, tcol, rows, c, s, idx, dz, K=None):
    """Eq. 10 for the given source rows j: g[j, t] = sum_{i in N^T(j), t < K[i]}
    c_i s_j dz[i, idx[j, t]]; (tptr, tcol) = CSR of the transpose."""
    k = idx.shape[1]
    out = np.zeros((rows.size, k))
    for r, j in enumerate(rows):
        dst = tcol[tptr[j]:tptr[j + 1]]
        for t in range(k):
            m = np.ones(dst.size, bool) if K is None else K[dst] > t
            out[r, t] = s[j] * np.sum(c[dst[m]] * dz[dst[m], idx[j, t]])
    return out


# ------------------------------------------------------------------ f2 at C4
def test_c4_ng_sampled_parity(c4):
    d = c4
    D, k = 128, 16
    thr, kb = (8, 32), (16, 8, 4)
    g = dr.Graph.from_design(d)
    rng = np.random.default_rng(3)
    for rel in ("near", "pins", "pinned"):
        ptr, col, nd, ns = (np.asarray(a) if i < 2 else a for i, a in enumerate(d.rel(rel)))
        x = d.x_net if rel == "pinned" else d.x_cell
        val, idx = dr.drelu_topk_sorted(cuda(x), k)
        oi, ov = to_np(idx).astype(np.int32), to_np(val).astype(np.float64)
        src_rows = _sample(ns, np.zeros(ns), rng)
        si, sv = O.drelu_sorted(x[src_rows].astype(np.float64), k)
        assert np.array_equal(oi[src_rows], si) and np.array_equal(ov[src_rows], sv), rel
        plan = dr.NgPlan(g, rel, thr, kb)
        z = to_np(dr.spmm_fwd_ng(plan, val, idx, D))
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        K = O.ng_k(ptr, thr, kb)
        deg = np.diff(ptr)
        hubs = np.nonzero(deg > 256)[0][:50]
        rows = _sample(nd, deg, rng, extra=hubs)
        assert row_err(z[rows], _fwd_rows(ptr, col, rows, c, s, oi, ov, D, K)) <= TOL, rel
        dz = rng.standard_normal((nd, D)).astype(np.float32)
        gk, _ = dr.spmm_bwd_ng(plan, cuda(dz), val, idx, D)
        tptr, tcol = (np.asarray(a) for a in d.rel(TRANSPOSE[rel])[:2])
        srows = _sample(ns, np.diff(tptr), rng)
        ref = _bwd_rows(tptr, tcol, srows, c, s, oi, dz.astype(np.float64), K)
        got = to_np(gk)[srows]
        # rows whose only surviving positions are single cancelling sums: the
        # summation-order bound (see tests/test_gpu_ng.py::within_cond)
        absr = _bwd_rows(tptr, tcol, srows, np.abs(c), np.abs(s), oi, np.abs(dz.astype(np.float64)), K)
        n_terms = np.diff(tptr)[srows]
        norms = np.linalg.norm(ref, axis=1, keepdims=True)
        bound = TOL * np.maximum(norms, 1e-30) + (n_terms[:, None] + 1) * 2.0 ** -24 * absr
        assert np.all(np.abs(got - ref) <= bound), rel


# ------------------------------------------------------------------ f3 at C2
def test_c2_full_per_edge_k_layer():
    d = make_config("C2")
    D, k, kp = 64, 8, 4
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 1, seed=7)
    W = {kk.split(".", 1)[1]: cuda(v) for kk, v in P.items() if kk.startswith("l0.")}
    L = dr.Layer(W, D, D, D, k, k, k_pins=kp)
    Wo = O.layer_params(P, 0)
    xc, xn = cuda(d.x_cell), cuda(d.x_net)
    yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn, flags=dr.DR_FWD_TAPS)
    v = dr.tape_view(g, L, tape, dr.DR_FWD_TAPS)
    T = {}
    for key, x, kk in (("hc", d.x_cell, k), ("hp", d.x_cell, kp), ("hn", d.x_net, k)):
        oi, ov = O.drelu(x.astype(np.float64), kk)
        assert np.array_equal(to_np(v[key + "_idx"]).astype(np.int32), oi), key
        assert np.array_equal(to_np(v[key + "_val"]), ov.astype(np.float32)), key
        T[key + "_idx"], T[key + "_val"] = oi, ov
    T["Hc"] = O.densify(T["hc_idx"], T["hc_val"], D)
    T["Hn"] = O.densify(T["hn_idx"], T["hn_val"], D)
    G = O.OGraph(d)
    for r in ("near", "pins", "pinned"):
        T["z_" + r] = to_np(v["z_" + r]).astype(np.float64)
    assert row_err(T["z_pins"], G.fwd("pins", T["hp_idx"], T["hp_val"], D)) <= TOL
    assert row_err(to_np(yn), T["z_pins"] @ Wo["wn_pins"] + T["Hn"] @ Wo["wr_pins"] + Wo["b_pins"]) <= TOL
    ta, tb = to_np(v["y_near"]), to_np(v["y_pinned"])
    T.update(M=ta >= tb, d_c=D, d_n=D, merge="max", root=True)
    rng = np.random.default_rng(5)
    dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
    dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
    grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, cuda(dyc), cuda(dyn), need_dx=True,
                                        flags=dr.DR_FWD_TAPS)
    og, odxc, odxn = O.layer_bwd(G, Wo, T, dyc, dyn, need_dx=True)
    for key in og:
        assert row_err(to_np(grads[key]), og[key]) <= TOL, key
    assert row_err(to_np(dxc), odxc) <= TOL
    assert row_err(to_np(dxn), odxn) <= TOL


# ------------------------------------------------------------------ f4 at C4
def test_c4_shard_w8_parity(c4):
    d = c4
    D, k, W = 128, 16, 8
    g = dr.Graph.from_design(d)
    rng = np.random.default_rng(9)
    for rel in ("near", "pins", "pinned"):
        ptr, col, nd, ns = d.rel(rel)
        X = cuda(d.x_net if rel == "pinned" else d.x_cell)
        dZ = cuda(rng.standard_normal((nd, D)).astype(np.float32))
        val, idx = dr.drelu_topk(X, k)
        shards = [dr.Shard.from_design(d, rel, W, q) for q in range(W)]
        m = shards[0].max_src
        va = torch.zeros(W * m, k, device="cuda")
        ia = torch.zeros(W * m, k, device="cuda", dtype=torch.uint8)
        for q, sh in enumerate(shards):
            n = sh.src_end - sh.src_begin
            va[q * m:q * m + n] = val[sh.src_begin:sh.src_end]
            ia[q * m:q * m + n] = idx[sh.src_begin:sh.src_end]
        z = torch.cat([sh.spmm_fwd(va, ia, D) for sh in shards])
        gp = sum(sh.spmm_bwd(dZ[sh.dst_begin:sh.dst_end].contiguous(), va, ia, D) for sh in shards)
        gs = torch.cat([gp[q * m:q * m + sh.src_end - sh.src_begin] for q, sh in enumerate(shards)])
        z1 = dr.spmm_fwd(g, rel, val, idx, D)
        g1, _ = dr.spmm_bwd(g, rel, dZ, val, idx, D)
        assert row_err(to_np(z), to_np(z1).astype(np.float64)) <= 4e-5, rel
        assert row_err(to_np(gs), to_np(g1).astype(np.float64)) <= 4e-5, rel
        ptr, col = np.asarray(ptr), np.asarray(col)
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        oi, ov = to_np(idx).astype(np.int32), to_np(val).astype(np.float64)
        rows = _sample(nd, np.diff(ptr), rng)
        assert row_err(to_np(z)[rows], _fwd_rows(ptr, col, rows, c, s, oi, ov, D)) <= TOL, rel
        del shards
