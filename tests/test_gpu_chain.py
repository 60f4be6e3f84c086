"""Row a5: the next layer's D-ReLU fused into the projection epilogue
(dr_heteroconv_fwd_chain; Eq. 2-3, applied to a layer's output,
which is the next layer's input).

Teacher-forced: the fused CBSR must be bit-identical (indices, values, sign of
zero) to oracle.drelu of the GPU's own fp32 Y (the D-ReLU decision is taken in
the kernel's precision, on the kernel's output); the chained two-layer forward
and the training step (fused + dead last-layer Y_net skipped) must equal the
unfused ones exactly."""
import numpy as np
import pytest

from gen import make_config, make_params
from oracle import oracle as O

from parity_util import to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.fixture(scope="module")
def designs():
    return {
        "C1": make_config("C1"),
        "C2s": make_config("C2", scale=0.1),
        "C4s": make_config("C4", scale=0.01),
    }


def _layer(P, l, dc, dn, D, kc, kn, scale=None):
    W = {k.split(".", 1)[1]: cuda(v) for k, v in P.items() if k.startswith(f"l{l}.")}
    return dr.Layer(W, dc, dn, D, kc, kn), W


def _check_cbsr(view, y_cell, y_net, kc, kn):
    for (vi, vv, y, k) in ((view["hc_idx"], view["hc_val"], y_cell, kc),
                           (view["hn_idx"], view["hn_val"], y_net, kn)):
        oi, ov = O.drelu(to_np(y).astype(np.float64), k)
        assert np.array_equal(to_np(vi).astype(np.int32), oi)
        got = to_np(vv)
        assert np.array_equal(got, ov.astype(np.float32))
        assert np.array_equal(np.signbit(got), np.signbit(ov))


# (design, d_cell, d_net, D, k_cell, k_net, next k_cell, next k_net)
CASES = [("C1", 16, 16, 16, 4, 4, 4, 4), ("C2s", 64, 64, 64, 8, 8, 8, 8),
         ("C4s", 128, 128, 128, 16, 16, 16, 16), ("C2s", 64, 64, 64, 8, 8, 32, 4),
         ("C1", 32, 16, 32, 8, 4, 16, 8), ("C2s", 64, 64, 128, 8, 8, 2, 16),
         ("C1", 16, 16, 256, 4, 4, 32, 16)]     # cells: N=256 (G=2) unfused fallback


@pytest.mark.parametrize("name,dc,dn,D,kc,kn,kc2,kn2", CASES)
def test_fused_next_drelu_bitexact(designs, name, dc, dn, D, kc, kn, kc2, kn2):
    d = designs[name]
    g = dr.Graph.from_design(d)
    P = make_params(dc, dn, D, 2, seed=11)
    P2 = make_params(D, D, D, 2, seed=12)
    L1, _ = _layer(P, 0, dc, dn, D, kc, kn)
    L2, _ = _layer(P2, 1, D, D, D, kc2, kn2)
    rng = np.random.default_rng(7)
    xc = cuda(rng.standard_normal((d.n_cell, dc)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, dn)).astype(np.float32))
    yc, yn, tape, nt = dr.heteroconv_fwd_chain(g, L1, xc, xn, next_layer=L2)
    v2 = dr.tape_view(g, L2, nt)
    _check_cbsr(v2, yc, yn, kc2, kn2)
    # Y_SCRATCH: same CBSR, Y need not be written
    _, _, _, nt2 = dr.heteroconv_fwd_chain(g, L1, xc, xn, next_layer=L2, flags=dr.DR_FWD_Y_SCRATCH)
    w2 = dr.tape_view(g, L2, nt2)
    for key in ("hc_idx", "hc_val", "hn_idx", "hn_val"):
        assert torch.equal(v2[key], w2[key]), key
    # the chained layer-1 outputs equal the plain forward's
    yc0, yn0, _ = dr.heteroconv_fwd(g, L1, xc, xn)
    assert torch.equal(yc, yc0) and torch.equal(yn, yn0)
    # layer 2 on its tape's CBSR == layer 2 on the dense Y (its own D-ReLU)
    y2c, y2n, _, _ = dr.heteroconv_fwd_chain(g, L2, None, None, tape=nt2,
                                             flags=dr.DR_FWD_INPUT_IN_TAPE)
    y2c0, y2n0, _ = dr.heteroconv_fwd(g, L2, yc0, yn0)
    assert torch.equal(y2c, y2c0) and torch.equal(y2n, y2n0)


@pytest.mark.parametrize("D,k", [(16, 4), (64, 8), (64, 32), (128, 16), (96, 8)])
@pytest.mark.parametrize("kind", ["ties", "ulp", "zeros"])
def test_fused_next_drelu_ties(designs, D, k, kind):
    """Zero weights make every row's Y the (merged) bias vector: exact ties
    (tie -> lowest column), 1-ulp neighbours (equal truncated composite keys:
    the in-epilogue exact rerun) and +-0.0 (one key)."""
    d = designs["C2s"]
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 1, seed=3)
    rng = np.random.default_rng(D + k)
    for key in P:
        if not key.startswith("l0."):
            continue
        if key.startswith("l0.b_"):
            if kind == "ties":
                P[key] = rng.integers(-2, 3, size=P[key].shape).astype(np.float32)
            elif kind == "ulp":
                base = np.float32(0.75)
                steps = rng.integers(0, 4, size=P[key].shape)
                P[key] = np.array([np.float32(base + s * np.spacing(base)) for s in steps.ravel()],
                                  np.float32).reshape(P[key].shape)
            else:
                P[key] = np.where(rng.random(P[key].shape) < 0.5, -0.0, 0.0).astype(np.float32)
        else:
            P[key] = np.zeros_like(P[key])
    L1, _ = _layer(P, 0, D, D, D, 4, 4)
    L2, _ = _layer(P, 0, D, D, D, k, k)
    xc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    yc, yn, _, nt = dr.heteroconv_fwd_chain(g, L1, xc, xn, next_layer=L2)
    _check_cbsr(dr.tape_view(g, L2, nt), yc, yn, k, k)


@pytest.mark.parametrize("name,D,k", [("C1", 16, 4), ("C2s", 64, 8), ("C4s", 128, 16)])
def test_trainer_chain_and_dead_net_exact(designs, knob, name, D, k):
    """The training step with the fused D-ReLU and the skipped last-layer Y_net
    gives the same loss, gradient and Adam update as the unfused step."""
    d = designs[name]
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 2, seed=21)
    lab = cuda(d.labels)
    rng = np.random.default_rng(5)
    xc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    out = {}
    for chain, dead in ((0, 0), (1, 1), (1, 0), (0, 1)):
        knob("chain", chain, 1)
        knob("skip_dead_net", dead, 1)
        flat = cuda(dr.flatten_params(P, 2))
        tr = dr.Trainer(flat, 2, D, D, D, k, k)
        grad = torch.empty_like(flat)
        losses = []
        for _ in range(3):                        # eager, captured, replayed
            losses.append(tr.step(g, xc, xn, lab, grad_out=grad))
        out[(chain, dead)] = (losses, grad.clone(), flat.clone())
        tr.close()
    ref = out[(0, 0)]
    for key, (losses, grad, flat) in out.items():
        assert losses == ref[0], key
        assert torch.equal(grad, ref[1]), key          # -0.0 == +0.0 for the zero pins grads
        assert torch.equal(flat, ref[2]), key


def test_chain_errors(designs):
    d = designs["C1"]
    g = dr.Graph.from_design(d)
    P = make_params(16, 16, 16, 2, seed=1)
    L1, _ = _layer(P, 0, 16, 16, 16, 4, 4)
    L2, _ = _layer(make_params(32, 32, 32, 2, seed=2), 1, 32, 32, 32, 4, 4)
    xc = cuda(np.ones((d.n_cell, 16), np.float32))
    xn = cuda(np.ones((d.n_net, 16), np.float32))
    with pytest.raises(dr.DRError) as e:
        dr.heteroconv_fwd_chain(g, L1, xc, xn, next_layer=L2)
    assert e.value.status == 3
    with pytest.raises(dr.DRError) as e:
        dr.heteroconv_fwd(g, L1, xc, xn, flags=dr.DR_FWD_INPUT_IN_TAPE)
    assert e.value.status == 1
    Lp = dr.Layer(_layer(P, 1, 16, 16, 16, 4, 4)[1], 16, 16, 16, 4, 4, k_pins=8)
    with pytest.raises(dr.DRError) as e:
        dr.heteroconv_fwd_chain(g, L1, xc, xn, next_layer=Lp)
    assert e.value.status == 12


@pytest.mark.parametrize("name,D,k", [("C2s", 64, 8), ("C4s", 128, 16)])
def test_split_z_bit_identical(designs, knob, name, D, k):
    """Z stored as split bf16 rows (read by the projection and the MN-major dW
    kernel as ready operand tiles) gives bit-identical outputs and gradients to
    fp32 Z converted by each consumer (same rounding)."""
    d = designs[name]
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 1, seed=4)
    L, _ = _layer(P, 0, D, D, D, k, k)
    rng = np.random.default_rng(3)
    xc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    dyc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    dyn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    out = {}
    for zs in (0, 1):
        knob("z_split", zs, 1)
        yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn)
        v = dr.tape_view(g, L, tape)
        assert v["z_split"] == [zs, zs, zs]
        grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)
        out[zs] = (yc, yn, grads, dxc, dxn)
    a, b = out[0], out[1]
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    assert torch.equal(a[3], b[3]) and torch.equal(a[4], b[4])
    for key in a[2]:
        assert torch.equal(a[2][key], b[2][key]), key


@pytest.mark.parametrize("name,D,k", [("C1", 16, 4), ("C2s", 64, 8), ("C4s", 128, 16)])
def test_trainer_fused_head_matches_separate(designs, knob, name, D, k):
    """The linear head + MSE fused into the last cell projection's epilogue (Y_cell
    never stored) against the separate head kernels on the stored Y_cell: the
    same quantities summed in another fixed order -- loss and every gradient
    within 1e-6 relative (the oracle parity of the fused path is
    test_gpu_parity.py::test_train_*)."""
    from parity_util import row_err
    d = designs[name]
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 2, seed=23)
    rng = np.random.default_rng(6)
    xc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    lab = cuda(d.labels)
    out = {}
    for fuse in (0, 1):
        knob("head_fuse", fuse, 1)
        flat = cuda(dr.flatten_params(P, 2))
        tr = dr.Trainer(flat, 2, D, D, D, k, k)
        grad = torch.empty_like(flat)
        loss = tr.step(g, xc, xn, lab, grad_out=grad)
        out[fuse] = (loss, to_np(grad).astype(np.float64))
        tr.close()
    assert abs(out[0][0] - out[1][0]) <= 1e-6 * abs(out[0][0])
    g0 = dr.unflatten(out[0][1], 2, D, D, D)
    g1 = dr.unflatten(out[1][1], 2, D, D, D)
    for key in g0:
        a = np.atleast_2d(g0[key])
        b = np.atleast_2d(g1[key])
        assert row_err(b, a) <= 1e-5, key


@pytest.mark.parametrize("name,D,k", [("C1", 16, 4), ("C2s", 64, 8)])
def test_trainer_two_epilogue_warpgroups(designs, knob, name, D, k):
    """The 16-warp row-GEMM layout (knob tc2_ewg = 2: two epilogue warpgroups on
    alternate tiles, setmaxnreg budgets) against the default 10-warp one: every
    row's epilogue arithmetic is the same, only the fused head's per-warp partial
    sums are added over 8 warps instead of 4 -- loss and gradients within 1e-6 /
    1e-5 row-normalised."""
    from parity_util import row_err
    d = designs[name]
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 2, seed=29)
    rng = np.random.default_rng(8)
    xc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    lab = cuda(d.labels)
    out = {}
    for ewg in (1, 2, 0):
        knob("tc2_ewg", ewg, 1)
        flat = cuda(dr.flatten_params(P, 2))
        tr = dr.Trainer(flat, 2, D, D, D, k, k)
        grad = torch.empty_like(flat)
        loss = tr.step(g, xc, xn, lab, grad_out=grad)
        out[ewg] = (loss, to_np(grad).astype(np.float64))
        tr.close()
    for ewg in (2, 0):
        assert abs(out[ewg][0] - out[1][0]) <= 1e-6 * abs(out[1][0])
        g0 = dr.unflatten(out[1][1], 2, D, D, D)
        g1 = dr.unflatten(out[ewg][1], 2, D, D, D)
        for key in g0:
            assert row_err(np.atleast_2d(g1[key]), np.atleast_2d(g0[key])) <= 1e-5, key


@pytest.mark.parametrize("name,D,k", [("C2s", 64, 8), ("C2s", 64, 16)])
def test_dw_dual_bit_identical(designs, knob, name, D, k):
    """The near and pinned weight gradients in one dual-B reduce launch (one pass
    over dY and the merge mask, Eq. 12-13's complementary masks as two B operands)
    against the two separate launches: the same MN-major operands, stages and MMA
    sequence per group, so every weight and bias gradient is bit-identical; the
    layer's other outputs are untouched."""
    d = designs[name]
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 1, seed=41)
    L, _ = _layer(P, 0, D, D, D, k, k)
    rng = np.random.default_rng(12)
    xc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    xn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    dyc = cuda(rng.standard_normal((d.n_cell, D)).astype(np.float32))
    dyn = cuda(rng.standard_normal((d.n_net, D)).astype(np.float32))
    out = {}
    for dual in (0, 1):
        knob("dw_dual", dual, 1)
        yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn)
        grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)
        out[dual] = (grads, dxc, dxn)
    a, b = out[0], out[1]
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    for key in a[0]:
        assert torch.equal(a[0][key], b[0][key]), key
