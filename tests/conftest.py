import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtgcu.so")
    # The CPU checkers are test infrastructure; build them if missing (cheap, gcc only).
    if not os.path.exists(os.path.join(ROOT, "oracle", "libtgoracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference, reference_available
    if not reference_available():
        pytest.skip("reference build oracle/_ref absent")
    return Reference()


def load_golden(name):
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", name))
