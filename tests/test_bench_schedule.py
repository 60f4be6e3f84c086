"""Host logic of bench.py's data-parallel C5 workload (SURVEY §8(d) 'DP
throughput'): the per-step, per-rank batches are a deterministic partition of
the designs, disjoint across ranks, with per-rank edge counts balanced to
within 5 % (designs vary ~2x in size), and the expected-nnz estimate used to
pack them tracks the generated designs."""
import numpy as np

import bench
from gen.circuit import c5_expected_nnz, make_c5_set


def test_c5_schedule_partition_and_balance():
    for world in (1, 2, 4, 8):
        b1, specs = bench.c5_schedule(world, 4)
        b2, _ = bench.c5_schedule(world, 4)
        assert b1 == b2                                   # deterministic on every rank
        assert len(b1) == 100 // (world * 4)
        seen = [i for s in b1 for r in s for i in r]
        assert len(seen) == len(set(seen))                # each design once per epoch
        for s in b1:
            assert len(s) == world and all(len(r) >= 1 for r in s)
            loads = np.array([sum(c5_expected_nnz(specs[i]) for i in r) for r in s])
            assert loads.max() <= 1.05 * loads.mean()


def test_expected_nnz_tracks_generated_designs():
    ds = make_c5_set(n_designs=4, workers=1)
    b, specs = bench.c5_schedule(1, 4, n_designs=4)
    for i, graphs in enumerate(ds):
        real = sum(sum(g.nnz().values()) for g in graphs)
        assert abs(c5_expected_nnz(specs[i]) - real) <= 0.06 * real
