"""Pins for oracle D-ReLU (Eq. 2-3; CBSR P:229).

Independent checks: SPEC worked vectors (golden), a numpy lexsort full-sort
brute force, exactly-k / dominance / idempotence invariants, k = D
identity, crafted rows (ties, +-0, all-negative, all-equal)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_vectors.json")))


@pytest.mark.parametrize("case", GOLD["drelu"], ids=lambda c: c["cite"][:40])
def test_spec_vectors(case):
    x = np.array([case["x"]], dtype=np.float64)
    idx, val = O.drelu(x, case["k"])
    assert idx[0].tolist() == case["idx"]
    assert val[0].tolist() == case["val"]
    assert np.array_equal(np.signbit(val[0]), np.signbit(np.array(case["val"], dtype=np.float64)))
    assert val[0].min() == case["threshold"]          # Eq. 2: th = min(topk)


def brute_topk(x, k):
    """Full sort with the (-x, col) key via numpy lexsort — an independent route."""
    n, d = x.shape
    idx = np.empty((n, k), np.int64)
    for r in range(n):
        xr = x[r] + 0.0                                  # -0.0 -> +0.0 for ordering only
        order = np.lexsort((np.arange(d), -xr))
        idx[r] = np.sort(order[:k])
    return idx


@pytest.mark.parametrize("d,k", [(16, 4), (64, 8), (128, 16), (32, 1), (40, 40), (256, 64)])
def test_bruteforce_with_ties(d, k):
    rng = np.random.default_rng(d * 1000 + k)
    x = rng.integers(-3, 4, size=(300, d)).astype(np.float64)      # many exact ties
    x[::7] = rng.standard_normal((x[::7].shape[0], d))
    x[5] = 0.0
    x[6, ::2] = -0.0
    idx, val = O.drelu(x, k)
    assert np.array_equal(idx, brute_topk(x, k))
    assert np.array_equal(val, np.take_along_axis(x, idx, 1))


def test_invariants():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((500, 64))
    x[:50] = np.round(x[:50])                      # ties
    k = 8
    idx, val = O.drelu(x, k)
    # exactly k, strictly ascending, in range
    assert idx.shape == (500, k)
    assert np.all(np.diff(idx, axis=1) > 0) and idx.min() >= 0 and idx.max() < 64
    # dominance: kept v, dropped u => v > u or (v == u and kept index < dropped index)
    for r in range(500):
        kept = set(idx[r].tolist())
        for j in range(64):
            if j in kept:
                continue
            for t, i in enumerate(idx[r]):
                assert x[r, i] > x[r, j] or (x[r, i] == x[r, j] and i < j)
    # idempotence on support
    dense = O.densify(idx, val, 64)
    dense[dense == 0] = -np.inf                       # dropped entries below every kept one
    idx2, _ = O.drelu(dense, k)
    assert np.array_equal(idx, idx2)


def test_k_equals_d_identity():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((20, 24))
    idx, val = O.drelu(x, 24)
    assert np.array_equal(idx, np.tile(np.arange(24), (20, 1)))
    assert np.array_equal(val, x)


def test_crafted_rows():
    x = np.array([[1.0] * 8,                                  # all equal -> first k columns
                  [-5, -4, -3, -2, -1, -6, -7, -8],           # all negative: literal values
                  [0.0, -0.0, 0.0, -0.0, 1e-30, -1e-30, 0.0, 0.0]])
    idx, val = O.drelu(x, 3)
    assert idx[0].tolist() == [0, 1, 2]
    assert idx[1].tolist() == [2, 3, 4] and val[1].tolist() == [-3, -2, -1]
    assert idx[2].tolist() == [0, 1, 4]           # 1e-30 first, then the two lowest-index zeros
    assert np.signbit(val[2][1])                  # -0.0 kept verbatim


def test_bad_k():
    with pytest.raises(ValueError):
        O.drelu(np.zeros((2, 4)), 5)
    with pytest.raises(ValueError):
        O.drelu(np.zeros((2, 4)), 0)


def test_backward_scatter_golden():
    c = GOLD["drelu_backward"][0]
    dense = O.densify(np.array([c["idx"]]), np.array([c["g"]], dtype=np.float64), c["D"])
    assert dense[0].tolist() == c["dense"]
