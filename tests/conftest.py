import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

try:
    from hypothesis import HealthCheck, settings

    settings.register_profile("ci", deadline=None, max_examples=25,
                              suppress_health_check=[HealthCheck.too_slow])
    settings.load_profile("ci")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libqm1b_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_arrays():
    return np.load(os.path.join(GOLDEN_DIR, "golden_arrays.npz"))


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (test infrastructure): build oracle/_oracle.so on demand."""
    so = os.path.join(ROOT, "oracle", "_oracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle import port

    return port


@pytest.fixture(scope="session")
def md_host():
    """CPU build of the device integral math (tests/cpu_md)."""
    import ctypes

    so = os.path.join(ROOT, "tests", "cpu_md", "_md_host.so")
    if not os.path.exists(so):
        subprocess.run(["sh", os.path.join(ROOT, "tests", "cpu_md", "build.sh")], check=True)
    return ctypes.CDLL(so)


@pytest.fixture(scope="session")
def sto3g():
    from paper_2311_01135_b200 import load_basis

    return load_basis("sto-3g")


@pytest.fixture(scope="session")
def gpu_lib():
    """The CUDA library with a visible device; GPU tests fail loudly (no fallback) if absent."""
    from paper_2311_01135_b200 import _lib

    return _lib.load(require_device=True)
