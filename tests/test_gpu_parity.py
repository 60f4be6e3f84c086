"""GPU (sm_100a, libdr.so) vs fp64 oracle parity, stage by stage.

Teacher-forced protocol: every GPU stage is compared with the oracle stage fed
the GPU's own inputs to that stage (its fp32 X for D-ReLU, its CBSR for the
SpMM, its Z / CBSR / mask for the projections and the backward). D-ReLU indices
and values must be bit-identical, the merge mask bit-identical, everything else
within 1e-4 max row-normalised relative error (north_star)."""
import numpy as np
import pytest

from gen import make_config, make_design, make_params
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")

RELS = ("near", "pins", "pinned")
MOD = {"near": O.MEAN, "pins": O.MEAN, "pinned": O.SYM}


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.fixture(scope="module")
def designs():
    return {
        "C1": make_config("C1"),
        "C2s": make_config("C2", scale=0.1),           # 10k cells, hubs present
        "C4s": make_config("C4", scale=0.01),          # 10k cells, D=128, k=16, d_max 5e4
    }


# ------------------------------------------------------------------ D-ReLU
@pytest.mark.parametrize("dim,k", [(16, 4), (64, 8), (128, 16), (256, 32), (64, 1), (32, 32),
                                   (128, 64), (96, 8), (4, 2), (32, 2), (32, 8), (32, 16),
                                   (64, 2), (64, 4), (64, 16), (64, 32), (128, 4), (128, 8),
                                   (128, 32)])
def test_drelu_bitexact(dim, k):
    rng = np.random.default_rng(dim * 31 + k)
    x = rng.standard_normal((3000, dim)).astype(np.float32)
    x[:300] = rng.integers(-2, 3, size=(300, dim)).astype(np.float32)   # heavy ties
    x[300] = 0.0
    x[301, ::2] = -0.0
    x[302] = -1.0
    x[303] = np.float32(1e-38)
    x[304, : dim // 2] = -0.0
    xg = cuda(x)
    val, idx = dr.drelu_topk(xg, k)
    oi, ov = O.drelu(to_np(xg).astype(np.float64), k)
    assert np.array_equal(to_np(idx).astype(np.int32), oi)
    assert np.array_equal(to_np(val), ov.astype(np.float32))
    assert np.array_equal(np.signbit(to_np(val)), np.signbit(ov))


@pytest.mark.parametrize("dim,k", [(64, 8), (128, 16), (32, 4), (64, 32), (64, 2), (32, 16), (128, 4)])
def test_drelu_thread_per_row_matches_warp_kernel(dim, k, knob):
    """The thread-per-row network D-ReLU (composite keys truncated by log2(dim)
    bits, exact rerun when the (k+1)-th shares the k-th's truncated key) gives
    the warp-per-row kernel's output bit for bit, on rows built to hit the rerun:
    values one ulp apart around the threshold, duplicated values, and a tail of
    rows that is not a multiple of the 32-row staging group."""
    rng = np.random.default_rng(dim + 7 * k)
    n = 4133
    x = rng.standard_normal((n, dim)).astype(np.float32)
    for r in range(0, 600):                   # near-ties: neighbours of the k-th value
        row = np.sort(x[r])[::-1]
        t = row[k - 1]
        j = rng.choice(dim, size=3, replace=False)
        x[r, j[0]] = np.nextafter(t, np.float32(np.inf))
        x[r, j[1]] = np.nextafter(t, np.float32(-np.inf))
        x[r, j[2]] = t
    x[600:900] = np.round(x[600:900] * 2) / 2      # many exact duplicates
    xg = cuda(x)
    out = {}
    for mode in (0, 2):                       # 2: the network kernel for every supported shape
        knob("drelu_tpr", mode, 1)
        v, i = dr.drelu_topk(xg, k)
        vs, is_ = dr.drelu_topk_sorted(xg, k) if k <= 32 else (None, None)
        torch.cuda.synchronize()
        out[mode] = (to_np(v), to_np(i), None if vs is None else to_np(vs), None if is_ is None else to_np(is_))
    for a, b in zip(out[0], out[2]):
        if a is not None:
            assert np.array_equal(a, b)
    oi, ov = O.drelu(x.astype(np.float64), k)
    assert np.array_equal(out[2][1].astype(np.int32), oi)


def test_drelu_strided_rows():
    x = torch.randn(500, 80, device="cuda")
    v, i = dr.drelu_topk(x[:, :64], 8)
    oi, ov = O.drelu(to_np(x[:, :64]).astype(np.float64), 8)
    assert np.array_equal(to_np(i).astype(np.int32), oi)


def test_drelu_bad_k():
    x = torch.randn(10, 64, device="cuda")
    with pytest.raises(dr.DRError) as e:
        dr.drelu_topk(x, 6)          # not a power of two
    assert e.value.status == 2


# ------------------------------------------------------------------ SpMM forward / backward
def _graph(d, **kw):
    return dr.Graph.from_design(d, **kw)


def _cbsr_for(d, rel, D, k, seed):
    rng = np.random.default_rng(seed)
    n_src = d.rel(rel)[3]
    x = cuda(rng.standard_normal((n_src, D)).astype(np.float32))
    return dr.drelu_topk(x, k)


@pytest.mark.parametrize("name,D,k", [("C1", 16, 4), ("C2s", 64, 8), ("C2s", 64, 32),
                                      ("C4s", 128, 16), ("C2s", 128, 2), ("C2s", 32, 1)])
@pytest.mark.parametrize("flags", [0, 2])           # degree-binned order / identity order
def test_spmm_fwd_parity(designs, name, D, k, flags):
    d = designs[name]
    g = _graph(d, flags=flags)
    for rel in RELS:
        ptr, col, nd, ns = d.rel(rel)
        val, idx = _cbsr_for(d, rel, D, k, seed=hash((name, rel)) % 1000)
        z = dr.spmm_fwd(g, rel, val, idx, D)
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        ref = O.spmm_fwd(ptr, col, nd, c, s, to_np(idx).astype(np.int32),
                         to_np(val).astype(np.float64), D)
        assert row_err(to_np(z), ref) <= TOL, rel
        deg = np.diff(ptr)
        assert np.all(to_np(z)[deg == 0] == 0.0)


def test_spmm_fwd_weighted(designs):
    d = designs["C2s"]
    rng = np.random.default_rng(3)
    w = {r: rng.uniform(0.2, 3.0, size=d.rel(r)[1].size).astype(np.float32) for r in RELS}
    g = _graph(d, weights=w)
    for rel in RELS:
        ptr, col, nd, ns = d.rel(rel)
        val, idx = _cbsr_for(d, rel, 64, 8, seed=7)
        z = dr.spmm_fwd(g, rel, val, idx, 64)
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        ref = O.spmm_fwd(ptr, col, nd, c, s, to_np(idx).astype(np.int32),
                         to_np(val).astype(np.float64), 64, a=w[rel].astype(np.float64))
        assert row_err(to_np(z), ref) <= TOL, rel
        dz = cuda(rng.standard_normal((nd, 64)).astype(np.float32))
        gk, _ = dr.spmm_bwd(g, rel, dz, val, idx, 64)
        refg = O.spmm_bwd(ptr, col, nd, ns, c, s, to_np(idx).astype(np.int32),
                          to_np(dz).astype(np.float64), a=w[rel].astype(np.float64))
        assert row_err(to_np(gk), refg) <= TOL, rel


@pytest.mark.parametrize("name,D,k", [("C1", 16, 4), ("C2s", 64, 8), ("C4s", 128, 16),
                                      ("C2s", 64, 64), ("C2s", 128, 4)])
def test_spmm_bwd_parity(designs, name, D, k):
    d = designs[name]
    g = _graph(d)
    rng = np.random.default_rng(11)
    for rel in RELS:
        ptr, col, nd, ns = d.rel(rel)
        val, idx = _cbsr_for(d, rel, D, k, seed=5)
        dz = cuda(rng.standard_normal((nd, D)).astype(np.float32))
        gk, dx = dr.spmm_bwd(g, rel, dz, val, idx, D, want_g=True, want_dx=True)
        c, s = O.normalisers(ptr, col, nd, ns, MOD[rel])
        oi = to_np(idx).astype(np.int32)
        ref = O.spmm_bwd(ptr, col, nd, ns, c, s, oi, to_np(dz).astype(np.float64))
        assert row_err(to_np(gk), ref) <= TOL, rel
        dense = O.densify(oi, to_np(gk).astype(np.float64), D)
        assert np.array_equal(to_np(dx), dense.astype(np.float32)), rel     # exact scatter
        # accumulate mode adds into the kept positions only
        # (the accumulate path is the SIMT kernel, the plain one may be the tensor-core
        # tiled kernel: same values up to rounding, same support)
        dx2 = torch.ones_like(dx)
        dr.spmm_bwd(g, rel, dz, val, idx, D, want_g=False, accumulate=True, dx_out=dx2)
        got = to_np(dx2).astype(np.float64) - 1.0
        want = O.densify(oi, ref, D)
        bound = TOL * np.linalg.norm(want, axis=1, keepdims=True) + 3e-7   # + ulp(1.0) of the add
        assert np.all(np.abs(got - want) <= bound), rel
        off = O.densify(oi, np.ones_like(ref), D) == 0
        assert np.all(to_np(dx2)[off] == 1.0), rel


def test_spmm_adjoint_on_gpu(designs):
    """<fwd(H), dZ> == <val, bwd(dZ)> with both sides from the GPU."""
    d = designs["C2s"]
    g = _graph(d)
    rng = np.random.default_rng(2)
    for rel in RELS:
        nd = d.rel(rel)[2]
        val, idx = _cbsr_for(d, rel, 64, 8, seed=9)
        z = dr.spmm_fwd(g, rel, val, idx, 64)
        dz = cuda(rng.standard_normal((nd, 64)).astype(np.float32))
        gk, _ = dr.spmm_bwd(g, rel, dz, val, idx, 64)
        lhs = float((z.double() * dz.double()).sum())
        rhs = float((val.double() * gk.double()).sum())
        assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + 1.0)


def test_spmm_deterministic(designs):
    d = designs["C4s"]
    g = _graph(d)
    val, idx = _cbsr_for(d, "pins", 128, 16, seed=1)
    z1 = dr.spmm_fwd(g, "pins", val, idx, 128)
    z2 = dr.spmm_fwd(g, "pins", val, idx, 128)
    assert torch.equal(z1, z2)
    assert g.info()["hub_rows_dst"][1] > 0          # the CTA-per-row path was exercised


# ------------------------------------------------------------------ HeteroConv layer
def _layer(P, l, dc, dn, D, kc, kn, merge=0):
    W = {k.split(".", 1)[1]: cuda(v) for k, v in P.items() if k.startswith(f"l{l}.")}
    return dr.Layer(W, dc, dn, D, kc, kn, merge=merge), W


def _oracle_tape(view, d_c, d_n, merge="max"):
    hc_idx = to_np(view["hc_idx"]).astype(np.int32)
    hn_idx = to_np(view["hn_idx"]).astype(np.int32)
    hc_val = to_np(view["hc_val"]).astype(np.float64)
    hn_val = to_np(view["hn_val"]).astype(np.float64)
    return dict(hc_idx=hc_idx, hc_val=hc_val, hn_idx=hn_idx, hn_val=hn_val,
                Hc=O.densify(hc_idx, hc_val, d_c), Hn=O.densify(hn_idx, hn_val, d_n),
                z_near=to_np(view["z_near"]).astype(np.float64),
                z_pins=to_np(view["z_pins"]).astype(np.float64),
                z_pinned=to_np(view["z_pinned"]).astype(np.float64),
                d_c=d_c, d_n=d_n, merge=merge, root=True)


def _unpack_mask(words, D):
    w = words.astype(np.uint32)
    bits = (w[:, :, None] >> np.arange(32, dtype=np.uint32)[None, None, :]) & 1
    return bits.reshape(w.shape[0], -1)[:, :D].astype(bool)


# (design, d_cell, d_net, D, k_cell, k_net): square layers of C1/C2/C4 shapes, and
# first-layer shapes with d_cell != d_net != D (K chunks < 64, stacked dW groups,
# 256-wide dz+root accumulators)
HC_CASES = [("C1", 16, 16, 16, 4, 4), ("C2s", 64, 64, 64, 8, 8), ("C4s", 128, 128, 128, 16, 16),
            ("C2s", 128, 64, 64, 16, 8), ("C1", 32, 16, 32, 8, 4), ("C4s", 64, 128, 128, 8, 32)]


@pytest.mark.parametrize("name,dc,dn,D,kc,kn", HC_CASES)
@pytest.mark.parametrize("flags", [dr.DR_FWD_TAPS, dr.DR_FWD_TAPS | dr.DR_FWD_SEQUENTIAL])
def test_heteroconv_parity(designs, name, dc, dn, D, kc, kn, flags):
    d = designs[name]
    g = _graph(d)
    P = make_params(dc, dn, D, 1, seed=5)
    L, W = _layer(P, 0, dc, dn, D, kc, kn)
    Wo = O.layer_params(P, 0)
    rng = np.random.default_rng(4)
    xc = cuda(rng.standard_normal((d.n_cell, dc)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, dn)).astype(np.float32))
    yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn, flags=flags)
    v = dr.tape_view(g, L, tape, flags)
    # D-ReLU stage: bit-exact on the GPU's fp32 input
    oi, ov = O.drelu(to_np(xc).astype(np.float64), kc)
    assert np.array_equal(to_np(v["hc_idx"]).astype(np.int32), oi)
    assert np.array_equal(to_np(v["hc_val"]), ov.astype(np.float32))
    oi, ov = O.drelu(to_np(xn).astype(np.float64), kn)
    assert np.array_equal(to_np(v["hn_idx"]).astype(np.int32), oi)
    # SpMM stage on the GPU's CBSR
    T = _oracle_tape(v, dc, dn)
    G = O.OGraph(d)
    assert row_err(to_np(v["z_near"]), G.fwd("near", T["hc_idx"], T["hc_val"], dc)) <= TOL
    assert row_err(to_np(v["z_pins"]), G.fwd("pins", T["hc_idx"], T["hc_val"], dc)) <= TOL
    assert row_err(to_np(v["z_pinned"]), G.fwd("pinned", T["hn_idx"], T["hn_val"], dn)) <= TOL
    # projections on the GPU's Z and CBSR
    y_near = T["z_near"] @ Wo["wn_near"] + T["Hc"] @ Wo["wr_near"] + Wo["b_near"]
    y_pinned = T["z_pinned"] @ Wo["w_pinned"] + Wo["b_pinned"]
    y_net = T["z_pins"] @ Wo["wn_pins"] + T["Hn"] @ Wo["wr_pins"] + Wo["b_pins"]
    assert row_err(to_np(v["y_near"]), y_near) <= TOL
    assert row_err(to_np(v["y_pinned"]), y_pinned) <= TOL
    assert row_err(to_np(yn), y_net) <= TOL
    # merge: mask bit-identical to the GPU taps, Y_cell picks exactly
    M = _unpack_mask(to_np(v["mask"]).view(np.uint32), D)
    ta, tb = to_np(v["y_near"]), to_np(v["y_pinned"])
    assert np.array_equal(M, ta >= tb)                     # Eq. 14, ties -> near
    assert np.array_equal(to_np(yc), np.where(M, ta, tb))
    # backward on the GPU's tape
    T["M"] = M
    dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
    dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
    grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, cuda(dyc), cuda(dyn), need_dx=True,
                                        flags=flags)
    assert dxc.shape == (d.n_cell, dc) and dxn.shape == (d.n_net, dn)
    og, odxc, odxn = O.layer_bwd(G, Wo, T, dyc, dyn, need_dx=True)
    for key in og:
        assert row_err(to_np(grads[key]), og[key]) <= TOL, key
    assert row_err(to_np(dxc), odxc) <= TOL
    assert row_err(to_np(dxn), odxn) <= TOL
    # off-support entries of dX are exact zeros (D-ReLU mask gradient)
    assert np.all(to_np(dxc)[odxc == 0] == 0)


def test_heteroconv_streams_bitidentical(designs):
    d = designs["C2s"]
    g = _graph(d)
    P = make_params(64, 64, 64, 1, seed=6)
    L, W = _layer(P, 0, 64, 64, 64, 8, 8)
    xc = torch.randn(d.n_cell, 64, device="cuda")
    xn = torch.randn(d.n_net, 64, device="cuda")
    a = dr.heteroconv_fwd(g, L, xc, xn, flags=0)
    b = dr.heteroconv_fwd(g, L, xc, xn, flags=dr.DR_FWD_SEQUENTIAL)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    dyc = torch.randn(d.n_cell, 64, device="cuda")
    dyn = torch.randn(d.n_net, 64, device="cuda")
    ga = dr.heteroconv_bwd(g, L, a[2], dyc, dyn, flags=0)
    gb = dr.heteroconv_bwd(g, L, b[2], dyc, dyn, flags=dr.DR_FWD_SEQUENTIAL)
    for key in ga[0]:
        assert torch.equal(ga[0][key], gb[0][key]), key
    assert torch.equal(ga[1], gb[1]) and torch.equal(ga[2], gb[2])


# ------------------------------------------------------------------ training step
def _tie_free(seed0, n_cell=60, D=16, k=4):
    for seed in range(seed0, seed0 + 300):
        d = make_design("t", n_cell, seed, d_cell=D, d_net=D, near_mean=6.0, near_cap=16,
                        pins_mean=2.5, pins_dmax=12, n_net=n_cell // 2)
        P = make_params(D, D, D, 2, seed=seed)
        G = O.OGraph(d)
        ok = True
        hc, hn = d.x_cell, d.x_net
        for l in range(2):
            for X in (hc, hn):
                s = -np.sort(-np.asarray(X, np.float64), axis=1)
                if np.any(s[:, k - 1] - s[:, k] < 1e-4):
                    ok = False
            hc, hn, tape = O.layer_fwd(G, O.layer_params(P, l), hc, hn, k, k)
            if np.abs(tape["y_near"] - tape["y_pinned"]).min() < 1e-4:
                ok = False
        if ok:
            return d, P, G
    raise RuntimeError("no tie-free instance")


def test_train_step_parity():
    """Free-running 2-layer step on a tie-free instance: loss, mean gradient and
    the Adam update match the oracle."""
    D, k = 16, 4
    d, P, G = _tie_free(100, D=D, k=k)
    g = _graph(d)
    flat = cuda(dr.flatten_params(P, 2))
    tr = dr.Trainer(flat, 2, D, D, D, k, k)
    grad = torch.empty_like(flat)
    loss = tr.step(g, cuda(d.x_cell), cuda(d.x_net), cuda(d.labels), grad_out=grad)
    oloss, og, _ = O.model_fwd_bwd(G, P, 2, k, k, d.x_cell, d.x_net, d.labels)
    assert abs(loss - oloss) <= TOL * abs(oloss)
    gg = dr.unflatten(to_np(grad), 2, D, D, D)
    for key in og:
        ref = og[key] if og[key].ndim == 2 else og[key].reshape(1, -1)
        got = gg[key] if gg[key].ndim == 2 else gg[key].reshape(1, -1)
        assert row_err(got, ref) <= TOL, key
    # Adam step-1 parameters
    th0 = dr.flatten_params(P, 2).astype(np.float64)
    ogf = dr.flatten_params({kk: og[kk] for kk in og}, 2).astype(np.float64)
    th1, _, _ = O.adam(th0, ogf, np.zeros_like(th0), np.zeros_like(th0), 1)
    assert np.max(np.abs(to_np(flat) - th1)) <= 1e-6


def test_train_multi_step_loss_trajectory():
    D, k = 16, 4
    d, P, G = _tie_free(400, D=D, k=k)
    g = _graph(d)
    flat = cuda(dr.flatten_params(P, 2))
    tr = dr.Trainer(flat, 2, D, D, D, k, k, lr=1e-3)
    th = dr.flatten_params(P, 2).astype(np.float64)
    m = np.zeros_like(th)
    v = np.zeros_like(th)
    for step in range(1, 6):
        loss = tr.step(g, cuda(d.x_cell), cuda(d.x_net), cuda(d.labels))
        Pcur = dr.unflatten(th, 2, D, D, D)
        oloss, og, _ = O.model_fwd_bwd(G, Pcur, 2, k, k, d.x_cell, d.x_net, d.labels)
        assert abs(loss - oloss) <= 1e-4 * abs(oloss), step
        th, m, v = O.adam(th, dr.flatten_params(og, 2).astype(np.float64), m, v, step, lr=1e-3)
    assert np.max(np.abs(to_np(flat) - th)) <= 1e-5


def test_train_step_c2_runs_and_loss_decreases():
    d = make_config("C2", scale=0.2)
    g = _graph(d)
    P = make_params(64, 64, 64, 2, seed=1)
    flat = cuda(dr.flatten_params(P, 2))
    tr = dr.Trainer(flat, 2, 64, 64, 64, 8, 8, lr=1e-3)
    xc, xn, y = cuda(d.x_cell), cuda(d.x_net), cuda(d.labels)
    losses = [tr.step(g, xc, xn, y) for _ in range(30)]
    assert np.all(np.isfinite(losses))
    assert losses[-1] < losses[0]


# ------------------------------------------------------------------ tensor-core dense path
@pytest.mark.parametrize("name,dc,dn,D,kc,kn", HC_CASES)
def test_dense_tcgen05_matches_simt(designs, name, dc, dn, D, kc, kn, knob):
    """The tcgen05 2xbf16-split projections / dZ / dW agree with the SIMT fp32
    kernels (both are separately pinned to the oracle above) to 5e-5
    row-normalised: each split operand carries |x - hi - lo| <= 2^-18 |x| and the
    dropped lo*lo term <= 2^-18 |a||b|, so a product is within ~2^-16.4 = 1.1e-5
    relative, and dX stacks the dz GEMM, the SSpMM and the root term."""
    d = designs[name]
    g = _graph(d)
    # one tape feeds both backward paths: keep Z in fp32 (the SIMT kernels do not
    # read split Z; test_gpu_chain.py::test_split_z_bit_identical covers split Z)
    knob("z_split", 0, 1)
    P = make_params(dc, dn, D, 1, seed=8)
    L, W = _layer(P, 0, dc, dn, D, kc, kn)
    rng = np.random.default_rng(12)
    xc = cuda(rng.standard_normal((d.n_cell, dc)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, dn)).astype(np.float32))
    dyc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    dyn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    # forward: Y_near / Y_pinned / Y_net of both paths; the merge mask may differ
    # only on near-ties of Y_near and Y_pinned (the two paths round differently)
    fw = {}
    for mode in ("0", "1"):
        knob("dense_simt", int(mode), 0)
        yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn, flags=dr.DR_FWD_TAPS)
        v = dr.tape_view(g, L, tape, dr.DR_FWD_TAPS)
        torch.cuda.synchronize()
        fw[mode] = dict(tape=tape, yn=to_np(yn), ya=to_np(v["y_near"]), yb=to_np(v["y_pinned"]),
                        M=_unpack_mask(to_np(v["mask"]).view(np.uint32), D))
    for key in ("yn", "ya", "yb"):
        assert row_err(fw["0"][key], fw["1"][key]) <= 5e-5, key
    ya, yb = fw["1"]["ya"], fw["1"]["yb"]
    flip = fw["0"]["M"] != fw["1"]["M"]
    scale = np.linalg.norm(ya, axis=1, keepdims=True) + np.linalg.norm(yb, axis=1, keepdims=True)
    assert np.all(np.abs(ya - yb)[flip] <= 5e-5 * np.broadcast_to(scale, ya.shape)[flip])
    # backward: both paths on the same (tc2) tape
    outs = {}
    for mode in ("0", "1"):
        knob("dense_simt", int(mode), 0)
        grads, dxc, dxn = dr.heteroconv_bwd(g, L, fw["0"]["tape"], dyc, dyn, flags=dr.DR_FWD_TAPS)
        torch.cuda.synchronize()
        outs[mode] = dict(dxc=to_np(dxc), dxn=to_np(dxn), **{kk: to_np(vv) for kk, vv in grads.items()})
    for key in outs["0"]:
        assert row_err(outs["0"][key], outs["1"][key]) <= 5e-5, key


@pytest.mark.parametrize("name,dc,dn,D,kc,kn", [("C2s", 64, 64, 64, 8, 8), ("C4s", 128, 128, 128, 16, 16)])
def test_heteroconv_sum_merge_parity(designs, name, dc, dn, D, kc, kn):
    """Eq. 6 variant: Y_cell = Y_near + Y_pinned, no mask routing."""
    d = designs[name]
    g = _graph(d)
    P = make_params(dc, dn, D, 1, seed=6)
    L, W = _layer(P, 0, dc, dn, D, kc, kn, merge=dr.DR_MERGE_SUM)
    Wo = O.layer_params(P, 0)
    rng = np.random.default_rng(8)
    xc = cuda(rng.standard_normal((d.n_cell, dc)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, dn)).astype(np.float32))
    yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn, flags=dr.DR_FWD_TAPS)
    v = dr.tape_view(g, L, tape, dr.DR_FWD_TAPS)
    T = _oracle_tape(v, dc, dn, merge="sum")
    y_near = T["z_near"] @ Wo["wn_near"] + T["Hc"] @ Wo["wr_near"] + Wo["b_near"]
    y_pinned = T["z_pinned"] @ Wo["w_pinned"] + Wo["b_pinned"]
    assert row_err(to_np(yc), y_near + y_pinned) <= TOL
    dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
    dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
    grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, cuda(dyc), cuda(dyn), need_dx=True,
                                        flags=dr.DR_FWD_TAPS)
    og, odxc, odxn = O.layer_bwd(O.OGraph(d), Wo, T, dyc, dyn, need_dx=True)
    for key in og:
        assert row_err(to_np(grads[key]), og[key]) <= TOL, key
    assert row_err(to_np(dxc), odxc) <= TOL
    assert row_err(to_np(dxn), odxn) <= TOL


@pytest.mark.parametrize("dim,k", [(64, 8), (128, 16), (32, 4), (256, 32)])
def test_drelu_ulp_near_ties(dim, k):
    """values a few ulps apart (the fast path's truncated keys collide and the
    full-key rerun decides): still bit-exact to the oracle"""
    rng = np.random.default_rng(dim + k)
    base = np.float32(1.0) + rng.integers(0, 40, size=(2000, dim)).astype(np.float32) * np.float32(2.0 ** -23)
    sign = np.where(rng.random((2000, dim)) < 0.3, -1.0, 1.0).astype(np.float32)
    x = (base * sign).astype(np.float32)
    val, idx = dr.drelu_topk(cuda(x), k)
    oi, ov = O.drelu(x.astype(np.float64), k)
    assert np.array_equal(to_np(idx).astype(np.int32), oi)
    assert np.array_equal(to_np(val), ov.astype(np.float32))
