"""Shared fixtures.  `-m gpu` tests need a B200 and the built library; the
CPU suite (`-m "not gpu"`) covers the oracle, host logic and the ABI surface."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and lib/libpf_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def acceptance_video():
    from oracle.reference_port import Params, generate_video

    return generate_video(Params(), 100, 128, 128, (64.0, 64.0), 42)


@pytest.fixture(scope="session")
def c1_video():
    from oracle.reference_port import Params, generate_video

    return generate_video(Params(), 10, 128, 128, (64.0, 64.0), 42)


def have_reference() -> bool:
    return os.path.isdir(REFERENCE_SRC)
