import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libkpo.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REF, "schedfront"))


@pytest.fixture(scope="session")
def schedfront():
    """The unmodified reference package (baseline/_ref), used only as a checker."""
    if not have_reference():
        pytest.skip("reference not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import schedfront as sf

    return sf


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_17654_b200 import _lib

    _lib.load()  # fail loudly (not skip) if the library is missing on a GPU box
    return torch.device("cuda", 0)
