import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle

    return Oracle.get()


@pytest.fixture(scope="session")
def reference():
    from pyoracle import Reference, have_reference

    if not have_reference() and not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return Reference.get()
