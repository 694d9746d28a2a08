"""Shared test setup.

`-m "not gpu"` tests run on CPU (oracle vs golden vectors, host logic, ABI
surface); `-m gpu` tests are the parity tests proper and call the CUDA path
through libhbgpu's C ABI.  The oracle (oracle/) is imported only here, as the
checker.
"""

import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhbgpu.so")


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def cuda():
    if not has_cuda():
        pytest.skip("no CUDA device")
    from paper_1304_7654_b200 import native
    native.require_cuda()
    return True
