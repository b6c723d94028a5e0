"""Shared pytest setup: the ``gpu`` marker, import paths, and common helpers."""
from __future__ import annotations

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built _lodb200.so")


def _gpu_available() -> bool:
    try:
        from paper_2310_03567_b200 import _lib

        return _lib.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """Fail loudly (not skip) when a gpu-marked test runs without a device."""
    from paper_2310_03567_b200 import _lib

    _lib.require_device(0)
    return 0


# the staged reference suite runs in its own pytest process (test_ref_suite.py)
collect_ignore_glob = ["ref_suite/*"]


@pytest.fixture(autouse=True)
def _release_device_memory(request):
    """After each GPU test, collect unreachable trees (facade objects can sit
    in reference cycles until the cyclic GC runs) so their arenas and node
    tables go back before the next test allocates its own."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    import gc

    gc.collect()
    try:
        import torch

        if torch.cuda.is_available():
            torch.cuda.empty_cache()
    except Exception:
        pass
