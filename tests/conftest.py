import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(__file__))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def _have(path):
    return os.path.exists(path)


@pytest.fixture(scope="session")
def capi():
    import tjtest
    return tjtest.Capi(0)


@pytest.fixture(scope="session")
def ref_module():
    """The reference trijoin Python module built from /root/reference (oracle/_ref)."""
    import tjtest
    if not _have(os.path.join(tjtest.REF_PKG, "trijoin", "__init__.py")):
        pytest.skip("reference build (oracle/_ref) not available")
    sys.path.insert(0, tjtest.REF_PKG)
    import trijoin
    return trijoin


@pytest.fixture(scope="session")
def oracle_lib():
    import tjtest
    if not _have(tjtest.ORACLE_LIB):
        pytest.skip("C restatement oracle not built (make -C oracle restatement)")
    return tjtest.load_oracle()
