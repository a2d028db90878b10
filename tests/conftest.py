import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) CUDA device")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _cuda_devices() -> int:
    import paper_1908_00210_b200 as pi

    return pi.device_count()


def pytest_collection_modifyitems(config, items):
    if not any("gpu" in item.keywords for item in items):
        return
    try:
        n = _cuda_devices()
    except Exception:  # import failure surfaces in the tests themselves
        return
    if n == 0:
        skip = pytest.mark.skip(reason="no CUDA device visible (run under gpurun)")
        for item in items:
            if "gpu" in item.keywords:
                item.add_marker(skip)
