"""Every D-ReLU kernel variant (Eq. 2-3) is bit-exact against the
oracle on tie-heavy rows: the cooperative thread-per-row network at 1, 2 and 4
lanes per row (knob drelu_coop), the whole-row network unrolled or in rolled
chunks (knob tpr_stream), the warp-per-row kernels (knob drelu_tpr), and the
defaults, at the D / k the workloads use. Rows 402-409 hold 1-ulp neighbours,
whose truncated composite keys tie at the threshold: the exact rerun
(tpr_rerun) decides them."""
import numpy as np
import pytest

from oracle import oracle as O

from parity_util import to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

dr = pytest.importorskip("paper_2508_16769_b200")


@pytest.mark.parametrize("dim,k", [(128, 16), (128, 8), (128, 4), (64, 8), (64, 16), (64, 4)])
@pytest.mark.parametrize("coop,tpr,stream", [(1, 1, 0), (2, 1, 0), (4, 1, 0), (0, 1, 0), (0, 2, 0),
                                             (0, 2, 2), (0, 0, 0), (-2, 1, 1), (2, 1, 2), (4, 1, 2)])
def test_drelu_variants_bitexact(knob, dim, k, coop, tpr, stream):
    knob("drelu_coop", coop, -2)
    knob("drelu_tpr", tpr, 1)
    knob("tpr_stream", stream, 1)
    rng = np.random.default_rng(dim + 7 * k + coop)
    x = rng.standard_normal((5003, dim)).astype(np.float32)        # ragged tail of a 32-row group
    x[:400] = rng.integers(-2, 3, size=(400, dim)).astype(np.float32)
    x[400] = 0.0
    x[401, ::2] = -0.0
    x[402:410] = np.float32(0.75) + rng.integers(0, 3, size=(8, dim)).astype(np.float32) * np.spacing(np.float32(0.75))
    xg = torch.as_tensor(x).cuda()
    val, idx = dr.drelu_topk(xg, k)
    oi, ov = O.drelu(x.astype(np.float64), k)
    assert np.array_equal(to_np(idx).astype(np.int32), oi)
    assert np.array_equal(to_np(val), ov.astype(np.float32))
    assert np.array_equal(np.signbit(to_np(val)), np.signbit(ov))


@pytest.mark.parametrize("dim,k", [(64, 8), (128, 16), (64, 16)])
@pytest.mark.parametrize("coop,tpr,stream", [(0, 2, 0), (0, 2, 2), (2, 1, 0), (2, 1, 2), (-2, 1, 1)])
def test_drelu_rerun_tie_counts(knob, dim, k, coop, tpr, stream):
    """The exact rerun's two regimes (tpr_rerun): m tied elements at the k-th
    value with m = 2 .. 16 (ranked one by one) and m = 17 .. D (bisection). Each
    row holds k - 3 larger values and m copies of the threshold value (exact ties:
    the lowest columns win), the rest smaller; some copies are replaced by 1-ulp
    neighbours so the truncated keys tie but the full keys do not."""
    knob("drelu_coop", coop, -2)
    knob("drelu_tpr", tpr, 1)
    knob("tpr_stream", stream, 1)
    rng = np.random.default_rng(11 + dim + k)
    rows = []
    for m in [2, 3, 8, 15, 16, 17, 24, dim - (k - 3)]:
        for ulp in (False, True):
            x = rng.uniform(-3.0, -1.0, dim).astype(np.float32)
            cols = rng.permutation(dim)
            big, tie = cols[:k - 3], cols[k - 3:k - 3 + m]
            x[big] = rng.uniform(2.0, 3.0, k - 3).astype(np.float32)
            x[tie] = np.float32(1.25)
            if ulp:
                x[tie[::3]] = np.nextafter(np.float32(1.25), np.float32(2.0))
            rows.append(x)
    x = np.stack(rows)
    xg = torch.as_tensor(x).cuda()
    val, idx = dr.drelu_topk(xg, k)
    oi, ov = O.drelu(x.astype(np.float64), k)
    assert np.array_equal(to_np(idx).astype(np.int32), oi)
    assert np.array_equal(to_np(val), ov.astype(np.float32))
