"""Shared pytest configuration.

`-m "not gpu"` runs on any CPU box: the oracle against the reference's golden
vectors, the host-side logic, and the C-ABI symbol table.  `-m gpu` runs the
parity tests proper through the CUDA library on a B200.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running check")


def has_reference() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "mixserve"))


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
