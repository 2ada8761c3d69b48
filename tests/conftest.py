import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference oracle (oracle/_ref); built on demand when the sources exist."""
    from oracle import ref as r
    if not r.available() and os.path.isdir("/root/reference/proj/src"):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    if not r.available():
        pytest.skip("reference oracle not built (oracle/_ref)")
    return r


@pytest.fixture(scope="session")
def rs():
    from oracle import restate
    return restate


@pytest.fixture(scope="session")
def s2b():
    import paper_2207_09776_b200 as m
    return m


@pytest.fixture(scope="session")
def ctx(s2b):
    return s2b.Context(0)
