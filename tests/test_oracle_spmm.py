"""Pins for the oracle DR-SpMM forward (Eq. 5-7, Alg. 1) and SSpMM backward
(Eq. 10-11, Alg. 2), and the degree normalisers (Q12).

Independent routes: a dense numpy brute force with degrees recounted by
np.bincount; scipy.sparse for k = D; the adjoint identity <fwd(H), dZ> =
<val, bwd(dZ)>; constant features under MEAN are the identity
(north_star); d-regular graphs make SYM == MEAN; SPEC worked vectors."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from gen import make_config
from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_vectors.json")))


def rand_csr(rng, n_dst, n_src, density, with_empty=True):
    A = (rng.random((n_dst, n_src)) < density)
    if with_empty and n_dst > 2:
        A[1] = False                      # isolated destination
        A[:, 0] = False if n_src > 1 else A[:, 0]
    ptr = np.concatenate([[0], np.cumsum(A.sum(1))]).astype(np.int64)
    col = np.nonzero(A)[1].astype(np.int32)
    return A, ptr, col


def dense_norm(A, module, weights=None):
    """Â = diag(c) A_w diag(s) with degrees recounted from the 0/1 pattern."""
    din = np.maximum(A.sum(1), 1).astype(np.float64)
    dout = np.maximum(A.sum(0), 1).astype(np.float64)
    Aw = A.astype(np.float64) if weights is None else weights
    if module == O.MEAN:
        return Aw / din[:, None]
    return Aw / np.sqrt(din)[:, None] / np.sqrt(dout)[None, :]


def rand_cbsr(rng, n, d, k):
    x = rng.standard_normal((n, d))
    return O.drelu(x, k)


@pytest.mark.parametrize("module", [O.MEAN, O.SYM])
@pytest.mark.parametrize("shape", [(30, 30, 0.2), (17, 40, 0.1), (50, 9, 0.3)])
def test_fwd_dense_bruteforce(module, shape):
    n_dst, n_src, dens = shape
    rng = np.random.default_rng(n_dst * 7 + module)
    A, ptr, col = rand_csr(rng, n_dst, n_src, dens)
    d, k = 12, 3
    idx, val = rand_cbsr(rng, n_src, d, k)
    w = rng.uniform(0.5, 2.0, size=col.size)
    for weights in (None, w):
        c, s = O.normalisers(ptr, col, n_dst, n_src, module)
        z = O.spmm_fwd(ptr, col, n_dst, c, s, idx, val, d, a=weights)
        Wd = None
        if weights is not None:
            Wd = np.zeros((n_dst, n_src))
            Wd[np.repeat(np.arange(n_dst), np.diff(ptr)), col] = weights
        ref = dense_norm(A, module, Wd) @ O.densify(idx, val, d)
        assert np.allclose(z, ref, rtol=1e-12, atol=1e-13)
        assert np.all(z[1] == 0.0)                    # isolated destination row -> 0


def test_fwd_k_equals_d_scipy():
    d = make_config("C1")
    ptr, col, nd, ns = d.rel("near")
    A = sp.csr_matrix((np.ones(col.size), col, ptr), shape=(nd, ns))
    x = d.x_cell.astype(np.float64)
    idx, val = O.drelu(x, x.shape[1])
    c, s = O.normalisers(ptr, col, nd, ns, O.MEAN)
    z = O.spmm_fwd(ptr, col, nd, c, s, idx, val, x.shape[1])
    deg = np.maximum(np.diff(ptr), 1)
    assert np.allclose(z, (A @ x) / deg[:, None], rtol=1e-12, atol=1e-14)


def test_constant_features_mean_is_identity():
    d = make_config("C1")
    ptr, col, nd, ns = d.rel("near")
    rng = np.random.default_rng(0)
    row = rng.standard_normal(16)
    x = np.tile(row, (ns, 1))
    idx, val = O.drelu(x, 4)
    c, s = O.normalisers(ptr, col, nd, ns, O.MEAN)
    z = O.spmm_fwd(ptr, col, nd, c, s, idx, val, 16)
    h = O.densify(idx[:1], val[:1], 16)[0]
    deg = np.diff(ptr)
    assert np.allclose(z[deg > 0], h, rtol=1e-14, atol=0)
    assert np.all(z[deg == 0] == 0.0)


def test_regular_graph_sym_equals_mean():
    n, r = 24, 4
    rows = np.repeat(np.arange(n), r)
    cols = (rows + np.tile(np.arange(1, r + 1), n)) % n        # circulant, in/out degree r
    ptr = np.arange(0, n * r + 1, r, dtype=np.int64)
    order = np.lexsort((cols, rows))
    col = cols[order].astype(np.int32)
    rng = np.random.default_rng(1)
    idx, val = rand_cbsr(rng, n, 8, 2)
    cm, sm = O.normalisers(ptr, col, n, n, O.MEAN)
    cs, ss = O.normalisers(ptr, col, n, n, O.SYM)
    zm = O.spmm_fwd(ptr, col, n, cm, sm, idx, val, 8)
    zs = O.spmm_fwd(ptr, col, n, cs, ss, idx, val, 8)
    assert np.allclose(zm, zs, rtol=1e-14, atol=1e-15)


def test_identity_adjacency():
    n = 10
    ptr = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    rng = np.random.default_rng(2)
    idx, val = rand_cbsr(rng, n, 6, 2)
    c, s = O.normalisers(ptr, col, n, n, O.SYM)
    z = O.spmm_fwd(ptr, col, n, c, s, idx, val, 6)
    assert np.array_equal(z, O.densify(idx, val, 6))
    dz = rng.standard_normal((n, 6))
    g = O.spmm_bwd(ptr, col, n, n, c, s, idx, dz)
    assert np.array_equal(g, O.gather_at(dz, idx))                  # S:263 identity gather


def test_spec_vectors():
    n = GOLD["spmm"][0]["n"]
    ptr = np.array([0, n], np.int64)
    col = np.arange(n, dtype=np.int32)
    ones = np.ones(1)
    z = O.spmm_fwd(ptr, col, 1, ones, np.ones(n), np.zeros((n, 1), np.int32), np.ones((n, 1)), 1)
    assert z[0, 0] == GOLD["spmm"][0]["y"]
    c2 = GOLD["spmm"][1]
    ptr = np.array([0, 2], np.int64)
    col = np.array([0, 1], np.int32)
    cc, ss = O.normalisers(ptr, col, 1, 2, O.MEAN)
    z = O.spmm_fwd(ptr, col, 1, cc, ss, np.array(c2["h_idx"], np.int32),
                   np.array(c2["h_val"]), c2["D"])
    assert z[0].tolist() == c2["z"]


@pytest.mark.parametrize("module", [O.MEAN, O.SYM])
def test_adjoint_identity(module):
    rng = np.random.default_rng(10 + module)
    A, ptr, col = rand_csr(rng, 40, 35, 0.15)
    w = rng.uniform(0.2, 3.0, size=col.size)
    d, k = 16, 5
    idx, val = rand_cbsr(rng, 35, d, k)
    c, s = O.normalisers(ptr, col, 40, 35, module)
    dz = rng.standard_normal((40, d))
    z = O.spmm_fwd(ptr, col, 40, c, s, idx, val, d, a=w)
    g = O.spmm_bwd(ptr, col, 40, 35, c, s, idx, dz, a=w)
    lhs = float((z * dz).sum())
    rhs = float((val * g).sum())
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


@pytest.mark.parametrize("module", [O.MEAN, O.SYM])
def test_bwd_masked_dense(module):
    rng = np.random.default_rng(20 + module)
    A, ptr, col = rand_csr(rng, 33, 27, 0.2)
    d, k = 10, 4
    idx, val = rand_cbsr(rng, 27, d, k)
    c, s = O.normalisers(ptr, col, 33, 27, module)
    dz = rng.standard_normal((33, d))
    g = O.spmm_bwd(ptr, col, 33, 27, c, s, idx, dz)
    full = dense_norm(A, module).T @ dz                       # (Â^T dZ), dense
    assert np.allclose(g, O.gather_at(full, idx), rtol=1e-12, atol=1e-13)
    # k = D reduces to the full transposed product (library routine)
    idxD, valD = rand_cbsr(rng, 27, d, d)
    gD = O.spmm_bwd(ptr, col, 33, 27, c, s, idxD, dz)
    As = sp.csr_matrix((np.ones(col.size), col, ptr), shape=(33, 27))
    An = sp.diags(c) @ As @ sp.diags(s)
    assert np.allclose(gD, An.T @ dz, rtol=1e-12, atol=1e-13)


def test_normalisers_against_bincount():
    d = make_config("C1")
    for r in ("near", "pins", "pinned"):
        ptr, col, nd, ns = d.rel(r)
        din = np.maximum(np.diff(ptr), 1)
        dout = np.maximum(np.bincount(col, minlength=ns), 1)
        c, s = O.normalisers(ptr, col, nd, ns, O.SYM)
        assert np.allclose(c, din ** -0.5, rtol=1e-15) and np.allclose(s, dout ** -0.5, rtol=1e-15)
        c, s = O.normalisers(ptr, col, nd, ns, O.MEAN)
        assert np.allclose(c, 1.0 / din, rtol=1e-15) and np.all(s == 1.0)
