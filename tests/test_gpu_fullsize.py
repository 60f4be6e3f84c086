"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (three relation streams, no taps), teacher-forced stage by stage
(SURVEY §8(c) P1):

* C2 (configs[1], 100k cells / 66.6k nets, D=64, k=8): every output of one
  HeteroConv layer forward + backward against the fp64 oracle fed the GPU's own
  inputs to each stage, plus the full 2-layer training step's loss.
* C4 (configs[3], 1M cells / 0.7M nets, D=128, k=16, hub nets of ~10^4 pins):
  the same, every row of every stage, through oracle.drelu / OGraph.fwd /
  numpy projections / oracle.layer_bwd fed the GPU's tape.

Bars: D-ReLU indices and values bit-exact; everything else <= 1e-4 max
row-normalised relative error (north_star). The merge decision M must equal
the oracle's [Y_near >= Y_pinned] wherever |Y_near - Y_pinned| exceeds 1e-5 of
the two row norms; closer near-ties are legitimately decided
by rounding, so they are counted, bounded (<= 1e-3 of all
elements) and checked only for validity (the GPU's Y_cell is one of the two
candidates)."""
import numpy as np
import pytest

from gen import make_config, make_params
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
dr = pytest.importorskip("paper_2508_16769_b200")


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _layer(P, D, k):
    W = {kk.split(".", 1)[1]: cuda(v) for kk, v in P.items() if kk.startswith("l0.")}
    return dr.Layer(W, D, D, D, k, k), O.layer_params(P, 0)


def _unpack_mask(words, D):
    w = words.astype(np.uint32)
    bits = (w[:, :, None] >> np.arange(32, dtype=np.uint32)[None, None, :]) & 1
    return bits.reshape(w.shape[0], -1)[:, :D].astype(bool)


GAP = 1e-5          # SURVEY §8(c) P2 near-tie band (fraction of the row norms)
MAX_TIES = 1e-3     # bound on the fraction of elements inside the band


def _merge_check(yc, M, y_near, y_pinned):
    """Eq. 8 / Eq. 14 merge on the oracle's Y_near / Y_pinned (fed the GPU's Z):
    the decision outside the near-tie band, the count of near-ties (bounded),
    validity inside it, and Y_cell against the GPU's own decision everywhere.
    Returns the number of near-tie elements."""
    scale = (np.linalg.norm(y_near, axis=1, keepdims=True) +
             np.linalg.norm(y_pinned, axis=1, keepdims=True))
    ok = np.abs(y_near - y_pinned) > GAP * scale
    assert np.array_equal(M[ok], (y_near >= y_pinned)[ok])
    n_tie = int((~ok).sum())
    assert n_tie <= MAX_TIES * ok.size, (n_tie, ok.size)
    yc = np.asarray(yc, np.float64)
    near_either = np.minimum(np.abs(yc - y_near), np.abs(yc - y_pinned)) <= TOL * scale
    assert np.all(near_either[~ok])
    assert row_err(yc, np.where(M, y_near, y_pinned)) <= TOL
    return n_tie


# ------------------------------------------------------------------ C2, every row
def test_c2_full_layer_parity():
    d = make_config("C2")
    D, k = 64, 8
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 1, seed=7)
    L, Wo = _layer(P, D, k)
    rng = np.random.default_rng(21)
    xc = cuda(d.x_cell)
    xn = cuda(d.x_net)
    yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn, flags=0)
    v = dr.tape_view(g, L, tape, 0)
    hc_idx, hn_idx = to_np(v["hc_idx"]).astype(np.int32), to_np(v["hn_idx"]).astype(np.int32)
    hc_val, hn_val = to_np(v["hc_val"]).astype(np.float64), to_np(v["hn_val"]).astype(np.float64)
    # D-ReLU: bit-exact on every row
    oi, ov = O.drelu(to_np(xc).astype(np.float64), k)
    assert np.array_equal(hc_idx, oi) and np.array_equal(to_np(v["hc_val"]), ov.astype(np.float32))
    oi, ov = O.drelu(to_np(xn).astype(np.float64), k)
    assert np.array_equal(hn_idx, oi) and np.array_equal(to_np(v["hn_val"]), ov.astype(np.float32))
    # SpMM on the GPU's CBSR, all rows
    G = O.OGraph(d)
    z = {r: to_np(v["z_" + r]).astype(np.float64) for r in ("near", "pins", "pinned")}
    assert row_err(z["near"], G.fwd("near", hc_idx, hc_val, D)) <= TOL
    assert row_err(z["pins"], G.fwd("pins", hc_idx, hc_val, D)) <= TOL
    assert row_err(z["pinned"], G.fwd("pinned", hn_idx, hn_val, D)) <= TOL
    # projections + merge on the GPU's Z / CBSR
    Hc, Hn = O.densify(hc_idx, hc_val, D), O.densify(hn_idx, hn_val, D)
    y_near = z["near"] @ Wo["wn_near"] + Hc @ Wo["wr_near"] + Wo["b_near"]
    y_pinned = z["pinned"] @ Wo["w_pinned"] + Wo["b_pinned"]
    assert row_err(to_np(yn), z["pins"] @ Wo["wn_pins"] + Hn @ Wo["wr_pins"] + Wo["b_pins"]) <= TOL
    M = _unpack_mask(to_np(v["mask"]).view(np.uint32), D)
    _merge_check(to_np(yc), M, y_near, y_pinned)
    # backward on the GPU's tape (mask included)
    dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
    dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
    grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, cuda(dyc), cuda(dyn), need_dx=True, flags=0)
    T = dict(hc_idx=hc_idx, hc_val=hc_val, hn_idx=hn_idx, hn_val=hn_val, Hc=Hc, Hn=Hn,
             z_near=z["near"], z_pins=z["pins"], z_pinned=z["pinned"], M=M, d_c=D, d_n=D,
             merge="max", root=True)
    og, odxc, odxn = O.layer_bwd(G, Wo, T, dyc, dyn, need_dx=True)
    for key in og:
        assert row_err(to_np(grads[key]), og[key]) <= TOL, key
    assert row_err(to_np(dxc), odxc) <= TOL
    assert row_err(to_np(dxn), odxn) <= TOL


def test_c2_full_train_step_loss():
    """The bench's training step on the full C2 design: the loss of step 1 equals
    the oracle's free-running 2-layer loss (near-tie rows are too few to move
    the mean beyond 1e-4)."""
    d = make_config("C2")
    D, k = 64, 8
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 2, seed=7)
    tr = dr.Trainer(cuda(dr.flatten_params(P, 2)), 2, D, D, D, k, k)
    loss = tr.step(g, cuda(d.x_cell), cuda(d.x_net), cuda(d.labels))
    oloss, _, _ = O.model_fwd_bwd(O.OGraph(d), P, 2, k, k, d.x_cell, d.x_net, d.labels)
    assert abs(loss - oloss) <= 1e-4 * abs(oloss)


# ------------------------------------------------------------------ C4, every row
def test_c4_full_every_row_parity():
    d = make_config("C4")
    D, k = 128, 16
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 1, seed=7)
    L, Wo = _layer(P, D, k)
    rng = np.random.default_rng(44)
    xc, xn = cuda(d.x_cell), cuda(d.x_net)
    yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn, flags=0)
    v = dr.tape_view(g, L, tape, 0)
    hc_idx, hn_idx = to_np(v["hc_idx"]).astype(np.int32), to_np(v["hn_idx"]).astype(np.int32)
    hc_val, hn_val = to_np(v["hc_val"]).astype(np.float64), to_np(v["hn_val"]).astype(np.float64)
    # D-ReLU: bit-exact on every row of both node types
    oi, ov = O.drelu(d.x_cell.astype(np.float64), k)
    assert np.array_equal(hc_idx, oi) and np.array_equal(to_np(v["hc_val"]), ov.astype(np.float32))
    oi, ov = O.drelu(d.x_net.astype(np.float64), k)
    assert np.array_equal(hn_idx, oi) and np.array_equal(to_np(v["hn_val"]), ov.astype(np.float32))
    del oi, ov
    G = O.OGraph(d)
    # SpMM forward, every destination row (the near tiles at D=128, k=16, the
    # adaptive CTA split, the hub nets), on the GPU's CBSR
    z = {r: to_np(v["z_" + r]).astype(np.float64) for r in ("near", "pins", "pinned")}
    assert row_err(z["near"], G.fwd("near", hc_idx, hc_val, D)) <= TOL
    assert row_err(z["pins"], G.fwd("pins", hc_idx, hc_val, D)) <= TOL
    assert row_err(z["pinned"], G.fwd("pinned", hn_idx, hn_val, D)) <= TOL
    # projections + merge, every row, on the GPU's Z / CBSR
    Hc, Hn = O.densify(hc_idx, hc_val, D), O.densify(hn_idx, hn_val, D)
    y_near = z["near"] @ Wo["wn_near"] + Hc @ Wo["wr_near"] + Wo["b_near"]
    y_pinned = z["pinned"] @ Wo["w_pinned"] + Wo["b_pinned"]
    assert row_err(to_np(yn), z["pins"] @ Wo["wn_pins"] + Hn @ Wo["wr_pins"] + Wo["b_pins"]) <= TOL
    M = _unpack_mask(to_np(v["mask"]).view(np.uint32), D)
    _merge_check(to_np(yc), M, y_near, y_pinned)
    del y_near, y_pinned, yc, yn
    # backward, every row, through oracle.layer_bwd on the GPU's tape (mask included)
    dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
    dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
    grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, cuda(dyc), cuda(dyn), need_dx=True, flags=0)
    T = dict(hc_idx=hc_idx, hc_val=hc_val, hn_idx=hn_idx, hn_val=hn_val, Hc=Hc, Hn=Hn,
             z_near=z["near"], z_pins=z["pins"], z_pinned=z["pinned"], M=M, d_c=D, d_n=D,
             merge="max", root=True)
    og, odxc, odxn = O.layer_bwd(G, Wo, T, dyc, dyn, need_dx=True)
    for key in og:
        assert row_err(to_np(grads[key]), og[key]) <= TOL, key
    assert row_err(to_np(dxc), odxc) <= TOL
    assert row_err(to_np(dxn), odxn) <= TOL
