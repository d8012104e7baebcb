import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"
REFERENCE_TESTS = "/root/reference/pkg/tests"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "reference: needs /root/reference (builder container only)")


def has_reference() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def spotrl():
    """The unmodified reference package, imported read-only (builder container only)."""
    if not has_reference():
        pytest.skip("reference package not present (it does not travel to the GPU box)")
    for p in (REFERENCE_SRC, REFERENCE_TESTS):
        if p not in sys.path:
            sys.path.append(p)
    import spotrl as mod
    return mod
