import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")


def _built():
    from paper_2508_03611_b200 import native
    if not os.path.exists(native.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()


@pytest.fixture(scope="session")
def ref():
    """The reference itself (oracle/_ref/libblocksim_ref.so) — the parity checker."""
    from oracle.oracle import Reference
    return Reference()


@pytest.fixture(scope="session")
def c_oracle():
    from oracle.oracle import CRestatement
    return CRestatement()


@pytest.fixture(scope="session")
def ctx():
    _built()
    from paper_2508_03611_b200 import native
    return native.Context(0)
