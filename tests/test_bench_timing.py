"""Host logic of bench.py's timed loop (timed_steps): every step runs exactly
once and in order, each between its own pair of events, behind one spin kernel
and (N > 1) one barrier per chunk of 16, with the garbage collector off inside
and back on afterwards -- also when a step raises. Runs on CPU with a stand-in
for torch.cuda that records the order of the enqueued operations."""
import gc

import pytest

import bench


class _Ev:
    def __init__(self, log, n):
        self.log, self.n, self.t = log, n, None

    def record(self):
        self.t = len(self.log)
        self.log.append(("event", self.n))

    def elapsed_time(self, other):
        return float(other.t - self.t)


class _Cuda:
    def __init__(self, log):
        self.log, self.k = log, 0

    def Event(self, enable_timing=False):
        self.k += 1
        return _Ev(self.log, self.k)

    def synchronize(self):
        self.log.append(("sync",))

    def _sleep(self, cycles):
        self.log.append(("spin", cycles))


class _Torch:
    def __init__(self, log):
        self.cuda = _Cuda(log)


class _Flush:
    def __init__(self, log):
        self.log = log

    def zero_(self):
        self.log.append(("flush",))


@pytest.mark.parametrize("n,barrier", [(50, False), (50, True), (16, True), (3, False)])
def test_timed_steps_order_chunks_and_gc(n, barrier):
    log = []
    steps = []
    bars = []

    def step(i):
        steps.append(i)
        log.append(("step", i))

    ms = bench.timed_steps(_Torch(log), step, n, _Flush(log),
                           barrier=(lambda: bars.append(len(log))) if barrier else None)
    assert steps == list(range(n))
    chunks = (n + 15) // 16
    assert sum(1 for x in log if x[0] == "spin") == chunks
    assert len(bars) == (chunks if barrier else 0)
    # every step: flush, start event, the step, end event -- nothing else in between
    for i in range(n):
        at = log.index(("step", i))
        assert log[at - 2] == ("flush",) and log[at - 1][0] == "event" and log[at + 1][0] == "event"
    # each spin precedes its chunk's steps and follows the previous chunk's drain
    spins = [k for k, x in enumerate(log) if x[0] == "spin"]
    for c, k in enumerate(spins):
        assert log[k - 1] == ("sync",)
        assert log.index(("step", 16 * c)) > k
    assert ms == pytest.approx(2.0 * n)           # each step's events bracket exactly 2 records
    assert len(bench.timed_steps.last) == n
    assert gc.isenabled()


def test_timed_steps_reenables_gc_on_error():
    log = []

    def step(i):
        if i == 5:
            raise RuntimeError("boom")

    with pytest.raises(RuntimeError):
        bench.timed_steps(_Torch(log), step, 20, _Flush(log))
    assert gc.isenabled()
