import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: CPU test that takes >30 s")


def pytest_collection_modifyitems(config, items):
    # GPU tests must not silently pass on a CPU box: they are deselected by
    # -m "not gpu" and fail loudly (no fallback) if run without a GPU.
    pass
