import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def built():
    """Build (or reuse) the product library and the oracle; returns the package module."""
    import __graft_entry__ as g
    g.build()
    import paper_2511_15028_b200 as sb
    return sb


@pytest.fixture(scope="session")
def oracle(built):
    from tests import oracle_lib
    return oracle_lib.Oracle()
