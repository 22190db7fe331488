import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run on the GPU box")
    config.addinivalue_line("markers", "slow: full-size configs (minutes); opt in with PRGPU_FULL=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("PRGPU_FULL") == "1":
        return
    skip = pytest.mark.skip(reason="full-size config; set PRGPU_FULL=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)
