"""Shared fixtures. ``-m gpu`` tests need a B200; everything else runs on CPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libvfpi.so")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
