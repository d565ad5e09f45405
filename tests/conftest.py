import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU check")


def load_golden(name):
    with open(os.path.join(GOLD, name + ".json")) as f:
        return json.load(f)["data"]


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture(scope="session")
def mdg():
    import paper_1911_08963_b200 as m
    m.lib()
    return m


@pytest.fixture(scope="session")
def device(mdg):
    dev = mdg.Device(0)
    yield dev
    dev.close()
