import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    from oracle import bindings as B
    if not os.path.exists(B.PORT_SO):
        B.build()
    return B.port()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref), or skip where it was never built."""
    from oracle import bindings as B
    if not os.path.exists(B.REF_SO) and os.path.isdir(B.REF_SRC):
        B.build()
    r = B.ref()
    if r is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return r


@pytest.fixture(scope="session")
def golden():
    import json
    d = os.path.join(ROOT, "tests", "golden")

    def load(name):
        with open(os.path.join(d, name)) as f:
            return json.load(f)
    return load
