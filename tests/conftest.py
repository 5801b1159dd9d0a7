import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    return {n[:-5]: load_golden(n) for n in os.listdir(GOLDEN) if n.endswith(".json")}


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle.Oracle()


@pytest.fixture(scope="session")
def reference_lib():
    import oracle
    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return oracle.Reference()


@pytest.fixture(scope="session")
def qmcg():
    import paper_1205_0106_b200 as pkg
    from paper_1205_0106_b200 import build
    build.build()
    return pkg


@pytest.fixture(scope="session")
def ctx(qmcg):
    c = qmcg.Context(0)
    yield c
    c.close()
