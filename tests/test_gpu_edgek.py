"""Per-edge-type k (SURVEY §8 f3 variant, DESIGN reading Q27) on the GPU:
dr_layer.k_pins gives pins its own cell CBSR. Teacher-forced layer parity against
oracle.layer_fwd/layer_bwd(k_p=...) (D-ReLU bit-exact, everything else <= 1e-4
row-normalised), stream/sequential bit-identity, and a free-running training step
against oracle.model_fwd_bwd(k_p=...)."""
import numpy as np
import pytest

from gen import make_config, make_design, make_params
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.fixture(scope="module")
def designs():
    return {"C1": make_config("C1"), "C2s": make_config("C2", scale=0.1),
            "C4s": make_config("C4", scale=0.01)}


def _layer(P, dc, dn, D, kc, kn, kp):
    W = {k.split(".", 1)[1]: cuda(v) for k, v in P.items() if k.startswith("l0.")}
    return dr.Layer(W, dc, dn, D, kc, kn, k_pins=kp), W


CASES = [("C1", 16, 16, 16, 4, 4, 8), ("C2s", 64, 64, 64, 8, 8, 4), ("C2s", 64, 64, 64, 4, 8, 16),
         ("C4s", 128, 128, 128, 16, 16, 8), ("C2s", 64, 32, 64, 8, 4, 32)]


@pytest.mark.parametrize("name,dc,dn,D,kc,kn,kp", CASES)
@pytest.mark.parametrize("seq", [0, 1])
def test_heteroconv_per_edge_k_parity(designs, name, dc, dn, D, kc, kn, kp, seq):
    flags = dr.DR_FWD_TAPS | (dr.DR_FWD_SEQUENTIAL if seq else 0)
    d = designs[name]
    g = dr.Graph.from_design(d)
    P = make_params(dc, dn, D, 1, seed=9)
    L, _ = _layer(P, dc, dn, D, kc, kn, kp)
    Wo = O.layer_params(P, 0)
    rng = np.random.default_rng(kp * 7 + kc)
    xc = cuda(rng.standard_normal((d.n_cell, dc)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, dn)).astype(np.float32))
    yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn, flags=flags)
    v = dr.tape_view(g, L, tape, flags)
    xc64 = to_np(xc).astype(np.float64)
    for key, k in (("hc", kc), ("hp", kp)):
        oi, ov = O.drelu(xc64, k)
        assert np.array_equal(to_np(v[key + "_idx"]).astype(np.int32), oi), key
        assert np.array_equal(to_np(v[key + "_val"]), ov.astype(np.float32)), key
    oi, ov = O.drelu(to_np(xn).astype(np.float64), kn)
    assert np.array_equal(to_np(v["hn_idx"]).astype(np.int32), oi)
    G = O.OGraph(d)
    T = dict(hc_idx=to_np(v["hc_idx"]).astype(np.int32), hc_val=to_np(v["hc_val"]).astype(np.float64),
             hn_idx=to_np(v["hn_idx"]).astype(np.int32), hn_val=to_np(v["hn_val"]).astype(np.float64),
             hp_idx=to_np(v["hp_idx"]).astype(np.int32), hp_val=to_np(v["hp_val"]).astype(np.float64),
             d_c=dc, d_n=dn, merge="max", root=True)
    T["Hc"] = O.densify(T["hc_idx"], T["hc_val"], dc)
    T["Hn"] = O.densify(T["hn_idx"], T["hn_val"], dn)
    assert row_err(to_np(v["z_pins"]), G.fwd("pins", T["hp_idx"], T["hp_val"], dc)) <= TOL
    assert row_err(to_np(v["z_near"]), G.fwd("near", T["hc_idx"], T["hc_val"], dc)) <= TOL
    for r in ("near", "pins", "pinned"):
        T["z_" + r] = to_np(v["z_" + r]).astype(np.float64)
    y_net = T["z_pins"] @ Wo["wn_pins"] + T["Hn"] @ Wo["wr_pins"] + Wo["b_pins"]
    assert row_err(to_np(yn), y_net) <= TOL
    ta, tb = to_np(v["y_near"]), to_np(v["y_pinned"])
    M = ta >= tb
    assert np.array_equal(to_np(yc), np.where(M, ta, tb))
    T["M"] = M
    dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
    dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
    grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, cuda(dyc), cuda(dyn), need_dx=True,
                                        flags=flags)
    og, odxc, odxn = O.layer_bwd(G, Wo, T, dyc, dyn, need_dx=True)
    for key in og:
        assert row_err(to_np(grads[key]), og[key]) <= TOL, key
    assert row_err(to_np(dxc), odxc) <= TOL
    assert row_err(to_np(dxn), odxn) <= TOL
    # dX_c is zero exactly off the union of the two kept supports
    sup = (O.densify(T["hc_idx"], np.ones_like(T["hc_val"]), dc) +
           O.densify(T["hp_idx"], np.ones_like(T["hp_val"]), dc)) > 0
    assert np.all(to_np(dxc)[~sup] == 0)


def test_per_edge_k_equal_is_per_node_type(designs):
    """k_pins == k_cell (or 0) is bit-identical to the per-node-type layer."""
    d = designs["C2s"]
    g = dr.Graph.from_design(d)
    P = make_params(64, 64, 64, 1, seed=2)
    xc = torch.randn(d.n_cell, 64, device="cuda")
    xn = torch.randn(d.n_net, 64, device="cuda")
    dyc = torch.randn(d.n_cell, 64, device="cuda")
    dyn = torch.randn(d.n_net, 64, device="cuda")
    outs = []
    for kp in (0, 8):
        L, _ = _layer(P, 64, 64, 64, 8, 8, kp)
        yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn)
        gr, dxc, dxn = dr.heteroconv_bwd(g, L, tape, dyc, dyn)
        outs.append((yc, yn, dxc, dxn, gr))
    a, b = outs
    for i in range(4):
        assert torch.equal(a[i], b[i])
    for key in a[4]:
        assert torch.equal(a[4][key], b[4][key]), key


def test_per_edge_k_streams_bitidentical(designs):
    d = designs["C4s"]
    g = dr.Graph.from_design(d)
    P = make_params(128, 128, 128, 1, seed=3)
    L, _ = _layer(P, 128, 128, 128, 16, 16, 4)
    xc = torch.randn(d.n_cell, 128, device="cuda")
    xn = torch.randn(d.n_net, 128, device="cuda")
    a = dr.heteroconv_fwd(g, L, xc, xn, flags=0)
    b = dr.heteroconv_fwd(g, L, xc, xn, flags=dr.DR_FWD_SEQUENTIAL)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    dyc = torch.randn(d.n_cell, 128, device="cuda")
    dyn = torch.randn(d.n_net, 128, device="cuda")
    ga = dr.heteroconv_bwd(g, L, a[2], dyc, dyn, flags=0)
    gb = dr.heteroconv_bwd(g, L, b[2], dyc, dyn, flags=dr.DR_FWD_SEQUENTIAL)
    for key in ga[0]:
        assert torch.equal(ga[0][key], gb[0][key]), key
    assert torch.equal(ga[1], gb[1]) and torch.equal(ga[2], gb[2])


def _tie_free(seed0, D=16, ks=(4, 8)):
    for seed in range(seed0, seed0 + 400):
        d = make_design("t", 60, seed, d_cell=D, d_net=D, near_mean=6.0, near_cap=16,
                        pins_mean=2.5, pins_dmax=12, n_net=30)
        P = make_params(D, D, D, 2, seed=seed)
        G = O.OGraph(d)
        ok = True
        hc, hn = d.x_cell, d.x_net
        for l in range(2):
            for X in (hc, hn):
                s = -np.sort(-np.asarray(X, np.float64), axis=1)
                for k in ks:
                    if np.any(s[:, k - 1] - s[:, k] < 1e-4):
                        ok = False
            hc, hn, tape = O.layer_fwd(G, O.layer_params(P, l), hc, hn, ks[0], ks[0], k_p=ks[1])
            if np.abs(tape["y_near"] - tape["y_pinned"]).min() < 1e-4:
                ok = False
        if ok:
            return d, P, G
    raise RuntimeError("no tie-free instance")


def test_train_step_per_edge_k_parity():
    D, k, kp = 16, 4, 8
    d, P, G = _tie_free(700, D=D, ks=(k, kp))
    g = dr.Graph.from_design(d)
    flat = cuda(dr.flatten_params(P, 2))
    tr = dr.Trainer(flat, 2, D, D, D, k, k, k_pins=kp)
    grad = torch.empty_like(flat)
    loss = tr.step(g, cuda(d.x_cell), cuda(d.x_net), cuda(d.labels), grad_out=grad)
    oloss, og, _ = O.model_fwd_bwd(G, P, 2, k, k, d.x_cell, d.x_net, d.labels, k_p=kp)
    assert abs(loss - oloss) <= TOL * abs(oloss)
    gg = dr.unflatten(to_np(grad), 2, D, D, D)
    for key in og:
        ref = og[key] if og[key].ndim == 2 else og[key].reshape(1, -1)
        got = gg[key] if gg[key].ndim == 2 else gg[key].reshape(1, -1)
        assert row_err(got, ref) <= TOL, key


def test_per_edge_k_no_nets():
    """A design whose pins / pinned relations are empty: the k_pins path still runs
    (pins' D-ReLU, an all-zero pins term) and matches the per-node-type layer."""
    d = make_config("C1")
    n_cell, n_net = d.n_cell, 1
    rels = {"near": d.rel("near")[:2], "pins": (np.zeros(n_net + 1, np.int64), np.zeros(0, np.int32)),
            "pinned": (np.zeros(n_cell + 1, np.int64), np.zeros(0, np.int32))}
    g = dr.Graph(n_cell, n_net, rels)
    P = make_params(16, 16, 16, 1, seed=4)
    xc = torch.randn(n_cell, 16, device="cuda")
    xn = torch.randn(n_net, 16, device="cuda")
    dyc = torch.randn(n_cell, 16, device="cuda")
    dyn = torch.randn(n_net, 16, device="cuda")
    outs = []
    for kp in (0, 8):
        L, _ = _layer(P, 16, 16, 16, 4, 4, kp)
        yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn)
        gr, dxc, dxn = dr.heteroconv_bwd(g, L, tape, dyc, dyn)
        outs.append((yc, yn, dxc, dxn))
    for a, b in zip(*outs):
        assert torch.allclose(a, b, rtol=0, atol=0)
