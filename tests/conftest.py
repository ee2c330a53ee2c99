import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def opts(request):
    """opts(ctx, name, value): nw_ctx_set_option for this test only (reset to the
    default, 0, when the test ends)."""
    undo = []

    def set_(ctx, name, value):
        ctx.set_option(name, value)
        undo.append((ctx, name))

    yield set_
    for ctx, name in reversed(undo):
        ctx.set_option(name, 0)
