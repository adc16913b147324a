import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libphfem_b200.so")


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    """The C oracle is test infrastructure; build it if the .so is missing."""
    so = os.path.join(ROOT, "oracle", "_build", "libphfem_oracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


@pytest.fixture(scope="session")
def ctx():
    from paper_2401_15557_b200 import capi
    c = capi.Context(0)
    yield c
    c.close()
