import os
import pathlib
import subprocess
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session", autouse=True)
def native_build():
    """Build (or no-op refresh) the native libraries, tests and oracles in-tree."""
    subprocess.run(["make", "-j8", "-C", str(REPO)], check=True, capture_output=True)
    subprocess.run(["make", "-C", str(REPO / "oracle"), "oracle"], check=True, capture_output=True)
    if pathlib.Path("/root/reference/proj").exists():
        subprocess.run(["make", "-j8", "-C", str(REPO / "oracle"), "ref"], check=True, capture_output=True)
    yield


@pytest.fixture(scope="session")
def gvx():
    import paper_2008_11476_b200 as m
    return m


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    return oracle


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(REPO / "tests" / "golden" / "configs.npz")
