import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size parity cases")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def _debug_guards(request):
    """DFC_DEBUG_GUARD=1: after every GPU test, check the canary zones around
    the outputs and the library's scratch allocations (tools/guard_run.sh)."""
    yield
    if os.environ.get("DFC_DEBUG_GUARD") == "1" and "gpu" in request.keywords:
        import paper_2106_03503_b200 as dfc
        dfc.check_guards()
