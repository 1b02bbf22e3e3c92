import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    # the checker library (oracle/) must exist for every test session
    if not os.path.exists(os.path.join(ROOT, "oracle", "libpms8oracle.so")):
        subprocess.run(["make", "c"], cwd=os.path.join(ROOT, "oracle"), check=True)


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gold():
    return golden
