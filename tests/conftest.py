"""Shared pytest plumbing.

Markers: ``gpu`` tests need a B200 (``-m gpu``); everything else runs on the
CPU build box (``-m "not gpu"``).  Golden fixtures live in tests/golden/.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


DECOMP_CASES = ["f1_dc", "f2_dc", "f1_256", "f1_thr", "const", "rand3", "rand11", "rand42",
                "atom", "c0", "c1", "c3_s0", "c3_s1", "big16384"]


@pytest.fixture(scope="session")
def golden():
    return load_golden
