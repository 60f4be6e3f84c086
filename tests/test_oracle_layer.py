"""Pins for the oracle HeteroConv layer, merge, head, Adam, 2-layer model and DP mean.

Independent routes:
  * k = D reduces the layer to textbook HeteroGraphConv{SAGEConv(mean),
    SAGEConv(mean), GraphConv(norm='both')} with aggregate=max; re-implemented
    here in dense torch fp64 with torch.autograd supplying the gradients;
  * central finite differences of the scalar loss (fp64, tie-free instances);
  * mask conservation / tie rule (Eq. 12-14); Adam against torch.optim.Adam;
  * DP mean of two equal-size batches == gradient over their disjoint union."""
import json
import os

import numpy as np
import pytest
import torch

from gen import disjoint_union, make_config, make_design, make_params
from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_vectors.json")))


def torch_dense_layer(design, W, x_c, x_n):
    """HeteroGraphConv with dense adjacency, k = D (no sparsification)."""
    def adj(r):
        ptr, col, nd, ns = design.rel(r)
        A = torch.zeros(nd, ns, dtype=torch.float64)
        A[torch.repeat_interleave(torch.arange(nd), torch.as_tensor(np.diff(ptr))),
          torch.as_tensor(col.astype(np.int64))] = 1.0
        return A
    An, Ap, Aq = adj("near"), adj("pins"), adj("pinned")
    mean = lambda A: A / A.sum(1, keepdim=True).clamp(min=1)
    sym = lambda A: A / A.sum(1, keepdim=True).clamp(min=1).sqrt() / A.sum(0, keepdim=True).clamp(min=1).sqrt()
    y_near = mean(An) @ x_c @ W["wn_near"] + x_c @ W["wr_near"] + W["b_near"]
    y_pinned = sym(Aq) @ x_n @ W["w_pinned"] + W["b_pinned"]
    y_net = mean(Ap) @ x_c @ W["wn_pins"] + x_n @ W["wr_pins"] + W["b_pins"]
    return torch.maximum(y_near, y_pinned), y_net


def test_layer_k_equals_d_matches_dense_torch():
    d = make_config("C1")
    P = make_params(16, 16, 16, 1, seed=3)
    G = O.OGraph(d)
    W = O.layer_params(P, 0)
    y_c, y_n, tape = O.layer_fwd(G, W, d.x_cell, d.x_net, 16, 16)
    Wt = {k: torch.tensor(v, requires_grad=True) for k, v in W.items()}
    xc = torch.tensor(d.x_cell.astype(np.float64), requires_grad=True)
    xn = torch.tensor(d.x_net.astype(np.float64), requires_grad=True)
    tc, tn = torch_dense_layer(d, Wt, xc, xn)
    assert np.allclose(y_c, tc.detach().numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(y_n, tn.detach().numpy(), rtol=1e-12, atol=1e-12)
    rng = np.random.default_rng(0)
    dyc, dyn = rng.standard_normal(y_c.shape), rng.standard_normal(y_n.shape)
    grads, dxc, dxn = O.layer_bwd(G, W, tape, dyc, dyn)
    (tc * torch.tensor(dyc)).sum().add((tn * torch.tensor(dyn)).sum()).backward()
    for k in W:
        assert np.allclose(grads[k], Wt[k].grad.numpy(), rtol=1e-10, atol=1e-12), k
    assert np.allclose(dxc, xc.grad.numpy(), rtol=1e-10, atol=1e-12)
    assert np.allclose(dxn, xn.grad.numpy(), rtol=1e-10, atol=1e-12)


def gaps_ok(x, k, thr):
    s = -np.sort(-x, axis=1)
    return np.all(s[:, k - 1] - s[:, k] > thr)


def tie_free_instance(seed0=1):
    """Redraw until every top-k gap and merge gap exceeds 1e-4 (SURVEY §8(c) O5 pin)."""
    for seed in range(seed0, seed0 + 200):
        d = make_design("fd", 40, seed, d_cell=16, d_net=16, near_mean=5.0, near_cap=16,
                        pins_mean=2.5, pins_dmax=12, n_net=25)
        P = make_params(16, 16, 16, 2, seed=seed)
        G = O.OGraph(d)
        if not (gaps_ok(d.x_cell, 4, 1e-3) and gaps_ok(d.x_net, 4, 1e-3)):
            continue
        ok = True
        hc, hn = d.x_cell, d.x_net
        for l in range(2):
            hc, hn, tape = O.layer_fwd(G, O.layer_params(P, l), hc, hn, 4, 4)
            if np.abs(tape["y_near"] - tape["y_pinned"]).min() < 1e-4:
                ok = False
            if l == 0 and not (gaps_ok(hc, 4, 1e-4) and gaps_ok(hn, 4, 1e-4)):
                ok = False
        if ok:
            return d, P, G
    raise RuntimeError("no tie-free instance")


def test_model_gradients_finite_differences():
    d, P, G = tie_free_instance()
    loss, grads, _ = O.model_fwd_bwd(G, P, 2, 4, 4, d.x_cell, d.x_net, d.labels)
    rng = np.random.default_rng(5)
    h = 1e-6
    checked = 0
    for name, arr in P.items():
        flat = arr.reshape(-1)
        for pos in rng.choice(flat.size, size=min(6, flat.size), replace=False):
            Pp = {k: v.astype(np.float64).copy() for k, v in P.items()}
            Pm = {k: v.astype(np.float64).copy() for k, v in P.items()}
            Pp[name].reshape(-1)[pos] += h
            Pm[name].reshape(-1)[pos] -= h
            lp = O.model_fwd_bwd(G, Pp, 2, 4, 4, d.x_cell, d.x_net, d.labels)[0]
            lm = O.model_fwd_bwd(G, Pm, 2, 4, 4, d.x_cell, d.x_net, d.labels)[0]
            fd = (lp - lm) / (2 * h)
            an = grads[name].reshape(-1)[pos]
            assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)) + 1e-9, (name, pos, fd, an)
            checked += 1
    assert checked > 50


def test_layer_input_gradient_finite_differences():
    d, P, G = tie_free_instance(50)
    W = O.layer_params(P, 1)                  # 16 -> 16 layer, inputs = features
    rng = np.random.default_rng(6)
    xc, xn = d.x_cell.astype(np.float64), d.x_net.astype(np.float64)
    y_c, y_n, tape = O.layer_fwd(G, W, xc, xn, 4, 4)
    dyc, dyn = rng.standard_normal(y_c.shape), rng.standard_normal(y_n.shape)
    _, dxc, dxn = O.layer_bwd(G, W, tape, dyc, dyn)

    def f(xc_, xn_):
        a, b, _ = O.layer_fwd(G, W, xc_, xn_, 4, 4)
        return float((a * dyc).sum() + (b * dyn).sum())
    h = 1e-6
    for (X, dX, which) in ((xc, dxc, 0), (xn, dxn, 1)):
        for _ in range(40):
            r, c = rng.integers(0, X.shape[0]), rng.integers(0, X.shape[1])
            Xp, Xm = X.copy(), X.copy()
            Xp[r, c] += h
            Xm[r, c] -= h
            fp = f(Xp, xn) if which == 0 else f(xc, Xp)
            fm = f(Xm, xn) if which == 0 else f(xc, Xm)
            fd = (fp - fm) / (2 * h)
            assert abs(fd - dX[r, c]) <= 1e-6 * max(1e-3, abs(dX[r, c])) + 1e-9


def test_merge_tie_rule_and_conservation():
    for case in GOLD["merge"]:
        yn, yp = np.array(case["y_near"]), np.array(case["y_pinned"])
        M = yn >= yp
        assert M.astype(int).tolist() == case["M"]
        assert np.where(M, yn, yp).tolist() == case["y"]
    d = make_config("C1")
    P = make_params(16, 16, 16, 1, seed=4)
    G = O.OGraph(d)
    W = O.layer_params(P, 0)
    _, _, tape = O.layer_fwd(G, W, d.x_cell, d.x_net, 4, 4)
    # isolated cell rows have Z = 0 in both relations -> Y_near vs Y_pinned decided by biases/root
    rng = np.random.default_rng(1)
    dyc = rng.standard_normal((d.n_cell, 16))
    M = tape["M"]
    dn, dp = np.where(M, dyc, 0.0), np.where(M, 0.0, dyc)
    assert np.array_equal(dn + dp, dyc)                    # bit-exact conservation


def test_zero_upstream_gives_zero_gradients():
    d = make_config("C1")
    P = make_params(16, 16, 16, 1, seed=4)
    G = O.OGraph(d)
    W = O.layer_params(P, 0)
    y_c, y_n, tape = O.layer_fwd(G, W, d.x_cell, d.x_net, 4, 4)
    grads, dxc, dxn = O.layer_bwd(G, W, tape, np.zeros_like(y_c), np.zeros_like(y_n))
    assert all(np.all(v == 0) for v in grads.values())
    assert np.all(dxc == 0) and np.all(dxn == 0)


def test_mse_golden_and_zero():
    c = GOLD["mse"][0]
    y = np.eye(2)
    pred = np.array([1.0, 0.0])                 # y = I, w_h = e_0, b_h = 0
    loss, g, dy = O.head_mse(y, np.array([1.0, 0.0]), np.array([0.0]),
                             pred - np.array(c["pred_minus_label"]))
    assert loss == c["loss"]
    assert dy[:, 0].tolist() == c["dpred"]
    loss0, g0, dy0 = O.head_mse(y, np.array([1.0, 2.0]), np.array([0.5]), np.array([1.5, 2.5]))
    assert loss0 == 0.0 and np.all(dy0 == 0)


def test_adam_matches_torch_and_closed_form():
    rng = np.random.default_rng(9)
    theta0 = rng.standard_normal(50)
    grads = [rng.standard_normal(50) for _ in range(5)]
    p = torch.tensor(theta0.copy(), requires_grad=True)
    opt = torch.optim.Adam([p], lr=2e-4, weight_decay=1e-5, betas=(0.9, 0.999), eps=1e-8)
    th, m, v = theta0.copy(), np.zeros(50), np.zeros(50)
    for t, g in enumerate(grads, 1):
        p.grad = torch.tensor(g)
        opt.step()
        th, m, v = O.adam(th, g, m, v, t)
        assert np.allclose(th, p.detach().numpy(), rtol=0, atol=1e-15)
    # step-1 closed form: update = -lr * g_hat / (|g_hat| + eps)
    gh = grads[0] + 1e-5 * theta0
    th1, _, _ = O.adam(theta0, grads[0], np.zeros(50), np.zeros(50), 1)
    assert np.allclose(th1 - theta0, -2e-4 * gh / (np.abs(gh) + 1e-8), rtol=1e-12, atol=1e-18)
    th0, _, _ = O.adam(theta0, grads[0], np.zeros(50), np.zeros(50), 1, lr=0.0)
    assert np.array_equal(th0, theta0)


def test_dp_mean_equals_union_gradient():
    a = make_design("a", 48, 11, d_cell=16, d_net=16, near_mean=5, near_cap=16, pins_mean=2.5,
                    pins_dmax=10, n_net=20)
    b = make_design("b", 48, 12, d_cell=16, d_net=16, near_mean=5, near_cap=16, pins_mean=2.5,
                    pins_dmax=10, n_net=30)
    P = make_params(16, 16, 16, 2, seed=2)
    ga = O.model_fwd_bwd(O.OGraph(a), P, 2, 4, 4, a.x_cell, a.x_net, a.labels)[1]
    gb = O.model_fwd_bwd(O.OGraph(b), P, 2, 4, 4, b.x_cell, b.x_net, b.labels)[1]
    u = disjoint_union([a, b])
    gu = O.model_fwd_bwd(O.OGraph(u), P, 2, 4, 4, u.x_cell, u.x_net, u.labels)[1]
    gm = O.dp_mean([ga, gb])
    for k in gu:
        assert np.allclose(gm[k], gu[k], rtol=1e-10, atol=1e-13), k


# ------------------------------------------------------------------ per-edge-type k (Q27, §8 f3)
def torch_topk_layer(design, W, x_c, x_n, k_c, k_p, k_n):
    """Independent route: D-ReLU as a torch.topk mask (tie-free instances), dense
    adjacency, autograd for the gradients. pins reads drelu(X_c, k_p), near and the
    near root drelu(X_c, k_c), pinned and the pins root drelu(X_n, k_n)."""
    def adj(r):
        ptr, col, nd, ns = design.rel(r)
        A = torch.zeros(nd, ns, dtype=torch.float64)
        A[torch.repeat_interleave(torch.arange(nd), torch.as_tensor(np.diff(ptr))),
          torch.as_tensor(col.astype(np.int64))] = 1.0
        return A

    def topk_mask(x, k):
        m = torch.zeros_like(x)
        m.scatter_(1, torch.topk(x.detach(), k, dim=1).indices, 1.0)
        return x * m
    An, Ap, Aq = adj("near"), adj("pins"), adj("pinned")
    mean = lambda A: A / A.sum(1, keepdim=True).clamp(min=1)
    sym = lambda A: A / A.sum(1, keepdim=True).clamp(min=1).sqrt() / A.sum(0, keepdim=True).clamp(min=1).sqrt()
    hc, hp, hn = topk_mask(x_c, k_c), topk_mask(x_c, k_p), topk_mask(x_n, k_n)
    y_near = mean(An) @ hc @ W["wn_near"] + hc @ W["wr_near"] + W["b_near"]
    y_pinned = sym(Aq) @ hn @ W["w_pinned"] + W["b_pinned"]
    y_net = mean(Ap) @ hp @ W["wn_pins"] + hn @ W["wr_pins"] + W["b_pins"]
    return torch.maximum(y_near, y_pinned), y_net


@pytest.mark.parametrize("k_c,k_p", [(4, 8), (8, 2), (4, 4)])
def test_layer_per_edge_type_k_matches_topk_autograd(k_c, k_p):
    for seed in range(1, 300):
        d = make_design("pe", 40, seed, d_cell=16, d_net=16, near_mean=5.0, near_cap=16,
                        pins_mean=2.5, pins_dmax=12, n_net=25)
        if all(gaps_ok(d.x_cell, k, 1e-3) for k in (k_c, k_p)) and gaps_ok(d.x_net, 4, 1e-3):
            break
    P = make_params(16, 16, 16, 1, seed=seed)
    G = O.OGraph(d)
    W = O.layer_params(P, 0)
    y_c, y_n, tape = O.layer_fwd(G, W, d.x_cell, d.x_net, k_c, 4, k_p=k_p)
    Wt = {k: torch.tensor(v, requires_grad=True) for k, v in W.items()}
    xc = torch.tensor(d.x_cell.astype(np.float64), requires_grad=True)
    xn = torch.tensor(d.x_net.astype(np.float64), requires_grad=True)
    tc, tn = torch_topk_layer(d, Wt, xc, xn, k_c, k_p, 4)
    assert np.allclose(y_c, tc.detach().numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(y_n, tn.detach().numpy(), rtol=1e-12, atol=1e-12)
    rng = np.random.default_rng(seed)
    dyc, dyn = rng.standard_normal(y_c.shape), rng.standard_normal(y_n.shape)
    grads, dxc, dxn = O.layer_bwd(G, W, tape, dyc, dyn)
    (tc * torch.tensor(dyc)).sum().add((tn * torch.tensor(dyn)).sum()).backward()
    for k in W:
        assert np.allclose(grads[k], Wt[k].grad.numpy(), rtol=1e-10, atol=1e-12), k
    assert np.allclose(dxc, xc.grad.numpy(), rtol=1e-10, atol=1e-12)
    assert np.allclose(dxn, xn.grad.numpy(), rtol=1e-10, atol=1e-12)


def test_layer_per_edge_type_k_reduces_to_per_node_type():
    """Y_cell depends on k_c only and Y_net on k_p only (near/pinned vs pins)."""
    d = make_config("C1")
    P = make_params(16, 16, 16, 1, seed=4)
    G = O.OGraph(d)
    W = O.layer_params(P, 0)
    yc, yn, _ = O.layer_fwd(G, W, d.x_cell, d.x_net, 4, 4, k_p=8)
    yc4, _, _ = O.layer_fwd(G, W, d.x_cell, d.x_net, 4, 4)
    _, yn8, _ = O.layer_fwd(G, W, d.x_cell, d.x_net, 8, 4)
    assert np.array_equal(yc, yc4)
    assert np.array_equal(yn, yn8)
