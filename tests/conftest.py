import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def corpus():
    with open(os.path.join(GOLDEN, "corpus.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def config_golden():
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    try:
        return Reference()
    except OSError:
        pytest.skip("oracle/_ref/libvcref.so not built (needs /root/reference at build time)")
