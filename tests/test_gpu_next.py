"""SURVEY §8 NEXT rows on the GPU: K-profiling (f1) returns a timed sweep and an
argmin per relation; the per-k paths it times agree with the oracle."""
import numpy as np
import pytest

from gen import make_config
from oracle import oracle as O

from parity_util import TOL, row_err, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")


def test_kprofile_sweep():
    from paper_2508_16769_b200.kprof import kprofile
    d = make_config("C2", scale=0.1)
    g = dr.Graph.from_design(d)
    rng = np.random.default_rng(0)
    xc = torch.as_tensor(rng.standard_normal((d.n_cell, 64)).astype(np.float32)).cuda()
    xn = torch.as_tensor(rng.standard_normal((d.n_net, 64)).astype(np.float32)).cuda()
    res = kprofile(g, xc, xn, ks=(2, 4, 8, 16, 32, 64, 128), reps=2)
    assert set(res) == {"near", "pins", "pinned"}
    for rel, r in res.items():
        assert set(r["times_ms"]) == {2, 4, 8, 16, 32, 64}           # k <= D only
        assert all(t > 0 for t in r["times_ms"].values())
        best = r["best_k"]
        assert r["times_ms"][best] == min(r["times_ms"].values())


@pytest.mark.parametrize("k", [2, 4, 32, 64])
def test_sweep_points_match_oracle(k):
    """every k the sweep visits runs a correct path (tiled where supported, SIMT else)"""
    d = make_config("C2", scale=0.1)
    g = dr.Graph.from_design(d)
    rng = np.random.default_rng(k)
    x = torch.as_tensor(rng.standard_normal((d.n_cell, 64)).astype(np.float32)).cuda()
    val, idx = dr.drelu_topk(x, k)
    z = dr.spmm_fwd(g, "near", val, idx, 64)
    ptr, col, nd, ns = d.rel("near")
    c, s = O.normalisers(ptr, col, nd, ns, O.MEAN)
    ref = O.spmm_fwd(ptr, col, nd, c, s, to_np(idx).astype(np.int32),
                     to_np(val).astype(np.float64), 64)
    assert row_err(to_np(z), ref) <= TOL
