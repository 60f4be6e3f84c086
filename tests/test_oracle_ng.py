"""Pins for the NEXT-2 (per-neighbour-group K) oracle functions, against things
other than themselves: a brute-force per-edge loop, the prefix property of the
value-sorted D-ReLU, the uniform-K reduction to the plain SpMM, the adjoint
identity and central finite differences."""
import numpy as np
import pytest

from gen import make_design
from oracle import oracle as O

pytestmark = pytest.mark.filterwarnings("ignore")


def _design():
    return make_design("ng", 300, 4, d_cell=16, d_net=16, near_mean=10.0, near_cap=40,
                       pins_mean=3.0, pins_dmax=30, n_net=200)


def test_drelu_sorted_prefix_is_topk():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((200, 16))
    x[:10, :8] = 1.0                                   # ties
    x[10:20] = 0.0
    idx, val = O.drelu_sorted(x, 8)
    for kk in range(1, 9):
        i2, v2 = O.drelu(x, kk)
        assert np.array_equal(np.sort(idx[:, :kk], axis=1), i2)      # same sets
    # value-descending, ties column-ascending, brute force
    for r in range(200):
        order = sorted(range(16), key=lambda c: (-x[r, c], c))[:8]
        assert list(idx[r]) == order
        assert np.array_equal(val[r], x[r, order])


def _brute_fwd(ptr, col, c, s, idx, val, d, K):
    z = np.zeros((len(ptr) - 1, d))
    for i in range(len(ptr) - 1):
        for e in range(ptr[i], ptr[i + 1]):
            j = col[e]
            for t in range(K[i]):
                z[i, idx[j, t]] += s[j] * val[j, t]
        z[i] *= c[i]
    return z


@pytest.mark.parametrize("rel", ["near", "pins", "pinned"])
def test_spmm_ng_brute_force_and_uniform(rel):
    d = _design()
    ptr, col, nd, ns = d.rel(rel)
    mod = O.SYM if rel == "pinned" else O.MEAN
    c, s = O.normalisers(ptr, col, nd, ns, mod)
    rng = np.random.default_rng(1)
    idx, val = O.drelu_sorted(rng.standard_normal((ns, 16)), 8)
    thr, kb = (3, 8), (8, 4, 2)
    K = O.ng_k(ptr, thr, kb)
    assert set(np.unique(K)) <= {8, 4, 2}
    z = O.spmm_fwd_ng(ptr, col, nd, c, s, idx, val, 16, thr, kb)
    assert np.allclose(z, _brute_fwd(ptr, col, c, s, idx, val, 16, K), rtol=1e-12, atol=1e-12)
    # uniform K = k: the plain SpMM (order inside a CBSR row does not matter)
    z8 = O.spmm_fwd_ng(ptr, col, nd, c, s, idx, val, 16, (10 ** 9, 10 ** 9), (8, 8, 8))
    assert np.allclose(z8, O.spmm_fwd(ptr, col, nd, c, s, idx, val, 16), rtol=1e-12, atol=1e-12)
    # every row in the last bin with K' = 4: the plain SpMM of the exact top-4 D-ReLU
    x = rng.standard_normal((ns, 16))
    i8, v8 = O.drelu_sorted(x, 8)
    i4, v4 = O.drelu(x, 4)
    z4 = O.spmm_fwd_ng(ptr, col, nd, c, s, i8, v8, 16, (-1, -1), (8, 8, 4))
    assert np.allclose(z4, O.spmm_fwd(ptr, col, nd, c, s, i4, v4, 16), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("rel", ["near", "pins"])
def test_spmm_ng_adjoint_and_fd(rel):
    d = _design()
    ptr, col, nd, ns = d.rel(rel)
    c, s = O.normalisers(ptr, col, nd, ns, O.MEAN)
    rng = np.random.default_rng(2)
    idx, val = O.drelu_sorted(rng.standard_normal((ns, 16)), 8)
    thr, kb = (4, 12), (8, 4, 2)
    dz = rng.standard_normal((nd, 16))
    z = O.spmm_fwd_ng(ptr, col, nd, c, s, idx, val, 16, thr, kb)
    g = O.spmm_bwd_ng(ptr, col, nd, ns, c, s, idx, dz, thr, kb)
    assert abs(np.sum(z * dz) - np.sum(val * g)) <= 1e-10 * (1 + abs(np.sum(z * dz)))
    # central finite differences of <Z(val), dz> w.r.t. a few CBSR values
    for (j, t) in [(0, 0), (5, 3), (17, 7), (ns - 1, 1)]:
        h = 1e-6
        vp, vm = val.copy(), val.copy()
        vp[j, t] += h
        vm[j, t] -= h
        fd = (np.sum(O.spmm_fwd_ng(ptr, col, nd, c, s, idx, vp, 16, thr, kb) * dz) -
              np.sum(O.spmm_fwd_ng(ptr, col, nd, c, s, idx, vm, 16, thr, kb) * dz)) / (2 * h)
        assert abs(fd - g[j, t]) <= 1e-6 * (1 + abs(fd))
