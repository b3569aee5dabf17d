"""Shared fixtures. `-m gpu` tests need a B200; everything else runs on CPU.

The CPU checkers (oracle/) are test infrastructure: built here on demand,
prebuilt .so files travel to GPU boxes with the repo snapshot.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    if not os.path.exists(O.ORACLE_SO) or (
            os.path.isdir(os.path.join(O.REF_SRC, "src")) and not os.path.exists(O.REF_SO)):
        O.build(ref=True)
    return O


@pytest.fixture(scope="session")
def lbgpu():
    import paper_1501_04741_b200 as P
    P.load_library()
    return P


@pytest.fixture(scope="session")
def has_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
