"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (three relation streams, no taps), teacher-forced stage by stage
(SURVEY §8(c) P1):

* C2 (configs[1], 100k cells / 66.6k nets, D=64, k=8): every output of one
  HeteroConv layer forward + backward against the fp64 oracle fed the GPU's own
  inputs to each stage, plus the full 2-layer training step's loss.
* C4 (configs[3], 1M cells / 0.7M nets, D=128, k=16, hub nets of ~10^4 pins):
  D-ReLU on every row; SpMM, projections, merge, SSpMM and dX on sampled rows
  (random, the heaviest rows, and every hub) which the oracle computes one by
  one from the GPU's tape; the weight gradients (full reductions over all rows)
  entirely.

Bars: D-ReLU indices and values bit-exact; everything else <= 1e-4 max
row-normalised relative error (north_star); the merge choice is checked where
the oracle's |Y_near - Y_pinned| gap exceeds 1e-4 of the row norm (closer ties
are legitimately decided by rounding)."""
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


def _gap_ok(y_near, y_pinned):
    """Rows/elements whose merge decision is not a near-tie."""
    scale = np.linalg.norm(y_near, axis=1, keepdims=True) + np.linalg.norm(y_pinned, axis=1, keepdims=True)
    return np.abs(y_near - y_pinned) > 1e-4 * scale


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
    ok = _gap_ok(y_near, y_pinned)
    assert np.array_equal(M[ok], (y_near >= y_pinned)[ok])
    assert row_err(np.where(ok, to_np(yc), 0.0), np.where(ok, np.where(M, y_near, y_pinned), 0.0)) <= TOL
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


# ------------------------------------------------------------------ C4, sampled rows
def _csr_rows(ptr, col, rows):
    """(edge dst position, neighbour id) of the given CSR rows."""
    starts, ends = ptr[rows], ptr[rows + 1]
    cnt = ends - starts
    pos = np.repeat(np.arange(rows.size), cnt)
    idx = np.concatenate([np.arange(s, e) for s, e in zip(starts, ends)]) if rows.size else np.zeros(0, np.int64)
    return pos, col[idx]


def _sample(n, deg, rng, extra=()):
    heavy = np.argsort(-deg, kind="stable")[:64]
    rnd = rng.choice(n, size=min(n, 3000), replace=False)
    return np.unique(np.concatenate([heavy, rnd, np.asarray(extra, np.int64)])).astype(np.int64)


def _spmm_rows(ptr, col, rows, c, s, hidx, hval, D):
    """Oracle Eq. 5 for the given destination rows only."""
    pos, nb = _csr_rows(ptr, col, rows)
    out = np.zeros((rows.size, D))
    k = hidx.shape[1]
    for t in range(k):
        np.add.at(out, (pos, hidx[nb, t]), s[nb] * hval[nb, t])
    return c[rows][:, None] * out


def test_c4_full_sampled_parity():
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
    G = O.OGraph(d)
    nptr, ncol = (np.asarray(a, np.int64) for a in d.rel("near")[:2])
    pptr, pcol = (np.asarray(a, np.int64) for a in d.rel("pins")[:2])       # nets -> cells
    qptr, qcol = (np.asarray(a, np.int64) for a in d.rel("pinned")[:2])     # cells -> nets
    cells = _sample(d.n_cell, np.diff(nptr), rng)
    hubs = np.nonzero(np.diff(pptr) > 256)[0]
    nets = _sample(d.n_net, np.diff(pptr), rng, extra=hubs)
    assert hubs.size > 0
    # SpMM forward on sampled destination rows (GPU CBSR as input)
    z_near = to_np(v["z_near"])
    z_pins = to_np(v["z_pins"])
    z_pinned = to_np(v["z_pinned"])
    c, s = G.cs["near"]
    assert row_err(z_near[cells], _spmm_rows(nptr, ncol, cells, c, s, hc_idx, hc_val, D)) <= TOL
    c, s = G.cs["pins"]
    assert row_err(z_pins[nets], _spmm_rows(pptr, pcol, nets, c, s, hc_idx, hc_val, D)) <= TOL
    c, s = G.cs["pinned"]
    assert row_err(z_pinned[cells], _spmm_rows(qptr, qcol, cells, c, s, hn_idx, hn_val, D)) <= TOL
    # projections + merge on sampled rows (GPU Z as input)
    Hc_s = O.densify(hc_idx[cells], hc_val[cells], D)
    Hn_s = O.densify(hn_idx[nets], hn_val[nets], D)
    y_near = z_near[cells].astype(np.float64) @ Wo["wn_near"] + Hc_s @ Wo["wr_near"] + Wo["b_near"]
    y_pinned = z_pinned[cells].astype(np.float64) @ Wo["w_pinned"] + Wo["b_pinned"]
    y_net = z_pins[nets].astype(np.float64) @ Wo["wn_pins"] + Hn_s @ Wo["wr_pins"] + Wo["b_pins"]
    assert row_err(to_np(yn)[nets], y_net) <= TOL
    Mw = to_np(v["mask"]).view(np.uint32)
    M_s = _unpack_mask(Mw[cells], D)
    ok = _gap_ok(y_near, y_pinned)
    assert np.array_equal(M_s[ok], (y_near >= y_pinned)[ok])
    assert row_err(np.where(ok, to_np(yc)[cells], 0.0), np.where(ok, np.where(M_s, y_near, y_pinned), 0.0)) <= TOL
    # backward on the GPU's tape
    dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
    dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
    grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, cuda(dyc), cuda(dyn), need_dx=True, flags=0)
    M = _unpack_mask(Mw, D)
    dy_near = np.where(M, dyc, 0.0)
    dy_pinned = np.where(M, 0.0, dyc)
    # weight gradients: full reductions over all rows
    Hc = _sparse_rows(hc_idx, hc_val, D)
    Hn = _sparse_rows(hn_idx, hn_val, D)
    ref = {"wn_near": z_near.T.astype(np.float64) @ dy_near, "wr_near": Hc.T @ dy_near,
           "b_near": dy_near.sum(0), "w_pinned": z_pinned.T.astype(np.float64) @ dy_pinned,
           "b_pinned": dy_pinned.sum(0), "wn_pins": z_pins.T.astype(np.float64) @ dyn,
           "wr_pins": Hn.T @ dyn.astype(np.float64), "b_pins": dyn.astype(np.float64).sum(0)}
    for key, r in ref.items():
        assert row_err(to_np(grads[key]), r) <= TOL, key
    # SSpMM + root term on sampled source rows (Alg. 2 / Eq. 10-11, oracle row by row)
    c_near, _ = G.cs["near"]
    c_pins, _ = G.cs["pins"]
    c_pinned, s_pinned = G.cs["pinned"]

    def dz_rows(dy, W, c, rows):
        return c[rows][:, None] * (dy[rows].astype(np.float64) @ W.T)

    # cells j: near (CSC = CSR, symmetric) + pins (CSC of pins = CSR of pinned: nets of j)
    g_c = np.zeros((cells.size, k))
    pos, nb = _csr_rows(nptr, ncol, cells)
    dzn = dz_rows(dy_near, Wo["wn_near"], c_near, nb)
    g_c += _sample_add(pos, dzn, hc_idx[cells], cells.size)
    pos, nb = _csr_rows(qptr, qcol, cells)
    dzp = dz_rows(dyn, Wo["wn_pins"], c_pins, nb)
    g_c += _sample_add(pos, dzp, hc_idx[cells], cells.size)
    g_c += np.take_along_axis(dy_near[cells] @ Wo["wr_near"].T, hc_idx[cells].astype(np.int64), 1)
    assert row_err(to_np(dxc)[cells], O.densify(hc_idx[cells], g_c, D)) <= TOL
    # nets j: pinned (CSC of pinned = CSR of pins: member cells of j), GraphConv s_j
    pos, nb = _csr_rows(pptr, pcol, nets)
    dzq = dz_rows(dy_pinned, Wo["w_pinned"], c_pinned, nb)
    g_n = s_pinned[nets][:, None] * _sample_add(pos, dzq, hn_idx[nets], nets.size)
    g_n += np.take_along_axis(dyn[nets].astype(np.float64) @ Wo["wr_pins"].T, hn_idx[nets].astype(np.int64), 1)
    assert row_err(to_np(dxn)[nets], O.densify(hn_idx[nets], g_n, D)) <= TOL


def _sample_add(pos, dz, idx_rows, n_rows):
    """sum over edges e of dz[e, idx_rows[pos[e], t]] into [n_rows, k]."""
    out = np.zeros((n_rows, idx_rows.shape[1]))
    vals = np.take_along_axis(dz, idx_rows[pos].astype(np.int64), axis=1)
    np.add.at(out, pos, vals)
    return out


def _sparse_rows(idx, val, D):
    import scipy.sparse as sp
    n, k = idx.shape
    return sp.csr_matrix((val.reshape(-1), idx.reshape(-1).astype(np.int64),
                          np.arange(0, n * k + 1, k, dtype=np.int64)), shape=(n, D))
