import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, TESTS):
    if _p not in sys.path:
        sys.path.insert(0, _p)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout at /root/reference")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "distsgd"))


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference package (imported in place, read-only)."""
    if not reference_available():
        pytest.skip("reference checkout not present (GPU box)")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import distsgd

    return distsgd
