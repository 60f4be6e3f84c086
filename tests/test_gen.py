"""Generator acceptance: determinism, structure and Table-1 ranges
 for CircuitNet-shaped graphs."""
import numpy as np

from gen import make_c5_set, make_config, make_design


def _csr_ok(ptr, col, n_rows, n_cols):
    assert ptr[0] == 0 and ptr[-1] == col.size and np.all(np.diff(ptr) >= 0)
    assert col.size == 0 or (col.min() >= 0 and col.max() < n_cols)
    for i in range(n_rows):
        seg = col[ptr[i]:ptr[i + 1]]
        assert np.all(np.diff(seg) > 0)


def test_c1_structure_and_crafted_cases():
    d = make_config("C1")
    _csr_ok(d.near_ptr, d.near_col, d.n_cell, d.n_cell)
    _csr_ok(d.pins_ptr, d.pins_col, d.n_net, d.n_cell)
    _csr_ok(d.pinned_ptr, d.pinned_col, d.n_cell, d.n_net)
    # near symmetric, no self loops
    A = np.zeros((d.n_cell, d.n_cell), bool)
    A[np.repeat(np.arange(d.n_cell), np.diff(d.near_ptr)), d.near_col] = True
    assert np.array_equal(A, A.T) and not A.diagonal().any()
    # pinned == pins^T
    B = np.zeros((d.n_net, d.n_cell), bool)
    B[np.repeat(np.arange(d.n_net), np.diff(d.pins_ptr)), d.pins_col] = True
    C = np.zeros((d.n_cell, d.n_net), bool)
    C[np.repeat(np.arange(d.n_cell), np.diff(d.pinned_ptr)), d.pinned_col] = True
    assert np.array_equal(B.T, C)
    nd, pd, qd = np.diff(d.near_ptr), np.diff(d.pins_ptr), np.diff(d.pinned_ptr)
    assert (nd == 0).any()                    # isolated cell
    assert (qd == 0).any()                    # cell in no net
    assert (pd == 1).any() and pd.max() == 16 and (pd == 0).any()   # 1-pin, hub, empty net
    assert (np.abs(d.x_cell).sum(1) == 0).any()                     # all-zero feature row


def test_determinism():
    a = make_design("x", 2000, 9, near_mean=20)
    b = make_design("x", 2000, 9, near_mean=20)
    for f in ("near_col", "pins_col", "pinned_col", "x_cell", "x_net", "labels"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_c5_table1_ranges():
    designs = make_c5_set(n_designs=2)
    for graphs in designs:
        assert 2 <= len(graphs) <= 4
        for g in graphs:
            near_mean = g.near_col.size / g.n_cell
            pins_per_net = g.pins_col.size / g.n_net
            assert 7300 <= g.n_cell < 9800
            assert 0.45 <= g.n_net / g.n_cell <= 0.95
            assert 34 <= near_mean <= 56, near_mean          # Table 1: 38-52 (+-10%)
            assert 1.9 <= pins_per_net <= 4.2, pins_per_net   # Table 1: 2.2-3.8 (+-10%)
            assert np.diff(g.near_ptr).max() <= 256
