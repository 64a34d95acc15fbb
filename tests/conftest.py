import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (B200); run with -m gpu")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def kat():
    return _load("kat.json")


@pytest.fixture(scope="session")
def random_suites():
    return _load("random_menus.json")


@pytest.fixture(scope="session")
def synthetic():
    return _load("synthetic.json")


@pytest.fixture(scope="session")
def orc():
    from oracle.pyoracle import ORC_PATH, Orc, build

    if not os.path.exists(ORC_PATH):
        build()
    return Orc()
