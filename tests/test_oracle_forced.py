"""Pins for the oracle's teacher-forcing helpers (reading Q28):
drelu_forced, drelu_gap, merge_gap and layer_fwd / model_fwd_bwd(forced=...).

Independent routes: per-row Python loops over the definition of a top-k
(every kept value >= every dropped value), forcing the oracle's own decisions
reproduces the free-running oracle bit for bit, and on all-equal rows every
selection is a valid top-k with value = the row's value."""
import numpy as np
import pytest

from gen import make_config, make_params
from oracle import oracle as O


def _gap_loops(x, idx):
    out = []
    for r in range(x.shape[0]):
        kept = set(int(c) for c in idx[r])
        kv = [x[r, c] for c in kept]
        dv = [x[r, c] for c in range(x.shape[1]) if c not in kept]
        nrm = float(np.sqrt(sum(v * v for v in x[r]))) or 1.0
        out.append((min(kv) - max(dv)) / nrm if dv else np.inf)
    return np.array(out)


def test_drelu_gap_against_loops():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((50, 16))
    idx, _ = O.drelu(x, 4)
    g = O.drelu_gap(x, idx)
    assert np.all(g >= 0)
    assert np.allclose(g, _gap_loops(x, idx))
    # swap the smallest kept column for the largest dropped one: a negative gap
    bad = idx.copy()
    for r in range(x.shape[0]):
        kept = list(idx[r])
        drop = [c for c in range(16) if c not in kept]
        kmin = min(kept, key=lambda c: x[r, c])
        dmax = max(drop, key=lambda c: x[r, c])
        kept[kept.index(kmin)] = dmax
        kept.sort()
        bad[r] = kept
    gb = O.drelu_gap(x, bad)
    assert np.all(gb < 0)
    assert np.allclose(gb, _gap_loops(x, bad))


def test_drelu_forced_own_selection_and_ties():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((40, 32))
    idx, val = O.drelu(x, 8)
    fi, fv = O.drelu_forced(x, idx)
    assert np.array_equal(fi, idx) and np.array_equal(fv, val)
    # all-equal rows: any ascending selection is a valid top-k
    xe = np.full((5, 8), 0.5)
    sel = np.array([[0, 1, 2], [5, 6, 7], [1, 3, 7], [0, 4, 6], [2, 3, 4]], np.int32)
    fi, fv = O.drelu_forced(xe, sel)
    assert np.all(fv == 0.5)
    assert np.all(O.drelu_gap(xe, sel) == 0)
    with pytest.raises(ValueError):
        O.drelu_forced(xe, sel[:, ::-1])             # not ascending
    with pytest.raises(ValueError):
        O.drelu_forced(xe, sel + 6)                  # out of range


def test_merge_gap_definition():
    rng = np.random.default_rng(2)
    a = rng.standard_normal((30, 12))
    b = rng.standard_normal((30, 12))
    M = a >= b
    assert np.all(O.merge_gap(a, b, M) >= 0)
    Mb = M.copy()
    Mb[3, 5] = ~Mb[3, 5]
    g = O.merge_gap(a, b, Mb)
    m = abs(a[3, 5] - b[3, 5]) / np.linalg.norm(np.maximum(a[3], b[3]))
    assert g[3] == pytest.approx(-m) or g[3] < -m + 1e-15
    assert np.all(np.delete(g, 3) >= 0)


def test_model_forced_with_own_decisions_is_free_running():
    d = make_config("C1")
    P = make_params(16, 16, 16, 2, seed=3)
    G = O.OGraph(d)
    loss, grads, tapes = O.model_fwd_bwd(G, P, 2, 4, 4, d.x_cell, d.x_net, d.labels)
    forced = [dict(hc_idx=t["hc_idx"], hn_idx=t["hn_idx"], M=t["M"]) for t in tapes]
    loss2, grads2, _ = O.model_fwd_bwd(G, P, 2, 4, 4, d.x_cell, d.x_net, d.labels, forced=forced)
    assert loss2 == loss
    for k in grads:
        assert np.array_equal(grads[k], grads2[k]), k


def test_model_forced_other_decisions_change_the_result():
    """Forcing a different (invalid) layer-2 selection changes the loss: the
    forced path really uses the given decisions."""
    d = make_config("C1")
    P = make_params(16, 16, 16, 2, seed=3)
    G = O.OGraph(d)
    loss, _, tapes = O.model_fwd_bwd(G, P, 2, 4, 4, d.x_cell, d.x_net, d.labels)
    alt = np.tile(np.arange(4, dtype=np.int32), (d.n_cell, 1))
    forced = [None, dict(hc_idx=alt)]
    loss2, _, tapes2 = O.model_fwd_bwd(G, P, 2, 4, 4, d.x_cell, d.x_net, d.labels, forced=forced)
    assert np.array_equal(tapes2[1]["hc_idx"], alt)
    assert loss2 != loss
