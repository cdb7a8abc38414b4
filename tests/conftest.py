import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def goldens():
    with open(os.path.join(HERE, "golden", "goldens.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from checkers import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from checkers import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libetwref.so not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def E():
    from paper_1709_09990_b200 import elimtw
    elimtw.library()
    return elimtw


@pytest.fixture(scope="session")
def gpu(E):
    info = E.device_info()
    if not info["available"]:
        pytest.fail("GPU test on a box without a usable CUDA device: " + str(info))
    return info


def instance_text(name):
    with open(os.path.join(HERE, "golden", "instances", name + ".gr")) as f:
        return f.read()


@pytest.fixture(scope="session")
def big_goldens():
    """Reference outputs for the large configs (tests/golden/make_big_goldens.py)."""
    with open(os.path.join(HERE, "golden", "big_goldens.json")) as f:
        return json.load(f)


def g48_golden():
    """The reference's full G(48,0.2) sweep (cfg 4, the bench workload), or
    None before tests/golden/make_big_goldens.py g48 has been run."""
    path = os.path.join(HERE, "golden", "g48_ref.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)
