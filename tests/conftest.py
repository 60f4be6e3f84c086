import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libdr.so")
    config.addinivalue_line("markers", "slow: larger CPU cases")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def knob():
    """Set a libdr experiment switch (dr_debug_set) for one test; restored after."""
    import paper_2508_16769_b200 as dr
    defaults = {}

    def set_(name, value, default):
        defaults.setdefault(name, default)
        dr.debug_set(name, value)
    yield set_
    for name, value in defaults.items():
        dr.debug_set(name, value)
