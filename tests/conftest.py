import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_2510_19225_b200  # noqa: E402,F401  (puts the installed reference `spotrl` on sys.path)

REFERENCE_TESTS = "/root/reference/pkg/tests"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "reference: needs /root/reference (builder container only)")


@pytest.fixture(scope="session")
def ref_tests():
    """The reference's own test directory (builder container only)."""
    if not os.path.isdir(REFERENCE_TESTS):
        pytest.skip("reference tests not present (they do not travel to the GPU box)")
    if REFERENCE_TESTS not in sys.path:
        sys.path.append(REFERENCE_TESTS)
    return REFERENCE_TESTS
