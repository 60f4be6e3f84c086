"""GPU checks of the dr_rel_desc optional inputs: a caller-supplied
CSC (Alg. 2 stage 1 "Transpose A to CSC") and caller degrees
give bit-identical results to the ones the library builds; caller normalisers
(c_i, s_j of Eq. 5 / Alg. 1) are the ones the SpMM and SSpMM apply, checked
against the fp64 oracle fed the same c and s."""
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
SRC = {"near": "cell", "pins": "cell", "pinned": "net"}


def _csc(ptr, col, n_src):
    rows = np.repeat(np.arange(ptr.size - 1, dtype=np.int64), np.diff(ptr))
    order = np.lexsort((rows, col))
    cptr = np.zeros(n_src + 1, np.int64)
    np.cumsum(np.bincount(col, minlength=n_src), out=cptr[1:])
    return cptr, rows[order].astype(np.int32)


@pytest.fixture(scope="module")
def design():
    return make_config("C2", scale=0.1)


def _run(g, d, D=64, k=8, seed=3):
    """D-ReLU + SpMM fwd + SSpMM bwd of every relation; outputs as numpy."""
    rng = np.random.default_rng(seed)
    out = {}
    x = {"cell": torch.as_tensor(rng.standard_normal((d.n_cell, D), dtype=np.float32)).cuda(),
         "net": torch.as_tensor(rng.standard_normal((d.n_net, D), dtype=np.float32)).cuda()}
    h = {t: dr.drelu_topk(x[t], k) for t in x}
    for r in RELS:
        val, idx = h[SRC[r]]
        z = dr.spmm_fwd(g, r, val, idx, D)
        dz = torch.as_tensor(rng.standard_normal(tuple(z.shape), dtype=np.float32)).cuda()
        gk, dx = dr.spmm_bwd(g, r, dz, val, idx, D, want_dx=True)
        out[r] = dict(z=to_np(z), g=to_np(gk), dx=to_np(dx), dz=to_np(dz),
                      idx=to_np(idx).astype(np.int32), val=to_np(val).astype(np.float64))
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("flags", [0, 1])      # 1 = DR_GRAPH_SKIP_VALIDATION: CSC used as given
def test_caller_csc_and_degrees_bit_identical(design, flags):
    d = design
    rels = {r: d.rel(r)[:2] for r in RELS}
    csc = {r: _csc(*d.rel(r)[:2], d.rel(r)[3]) for r in RELS}
    deg = {r: (np.diff(d.rel(r)[0]).astype(np.int32),
               np.bincount(d.rel(r)[1], minlength=d.rel(r)[3]).astype(np.int32)) for r in RELS}
    g0 = dr.Graph(d.n_cell, d.n_net, rels)
    g1 = dr.Graph(d.n_cell, d.n_net, rels, csc=csc, degrees=deg, flags=flags)
    assert g1.info()["tiles"] == g0.info()["tiles"]
    a, b = _run(g0, d), _run(g1, d)
    for r in RELS:
        for key in ("z", "g", "dx"):
            assert np.array_equal(a[r][key], b[r][key]), (r, key)


def test_caller_normalisers_and_degrees_match_oracle(design):
    """norm_dst / norm_src replace c / s; deg_dst / deg_src (e.g. the degrees of a
    larger design this graph is cut from) feed the module's formula (Q12)."""
    d = design
    rng = np.random.default_rng(11)
    rels = {r: d.rel(r)[:2] for r in RELS}
    norms = {"pinned": (rng.uniform(0.2, 1.5, d.n_cell).astype(np.float32),
                        rng.uniform(0.2, 1.5, d.n_net).astype(np.float32)),
             "near": (rng.uniform(0.01, 0.1, d.n_cell).astype(np.float32), None)}
    big = {"pins": (np.diff(d.rel("pins")[0]).astype(np.int32) + rng.integers(0, 5, d.n_net).astype(np.int32),
                    None)}
    g = dr.Graph(d.n_cell, d.n_net, rels, norms=norms, degrees=big)
    out = _run(g, d)
    for r in RELS:
        ptr, col, nd, ns = d.rel(r)
        c, s = O.normalisers(ptr, col, nd, ns, MOD[r])
        if r in norms:
            c = norms[r][0].astype(np.float64)
            if norms[r][1] is not None:
                s = norms[r][1].astype(np.float64)
        if r in big:               # MEAN: c_i = 1 / max(deg_i, 1) with the caller's degree
            c = (1.0 / np.maximum(big[r][0], 1)).astype(np.float32).astype(np.float64)
        o = out[r]
        ref_z = O.spmm_fwd(ptr, col, nd, c, s, o["idx"], o["val"], 64)
        ref_g = O.spmm_bwd(ptr, col, nd, ns, c, s, o["idx"], o["dz"].astype(np.float64))
        assert row_err(o["z"], ref_z) <= TOL, r
        assert row_err(o["g"], ref_g) <= TOL, r
