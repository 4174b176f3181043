import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libmmas.so")
    config.addinivalue_line("markers", "slow: long-running (still part of the default suite)")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # -m gpu tests are only skipped when explicitly deselected by the marker expression;
    # if they are selected on a box without a GPU they fail loudly (never a silent pass).
    pass
