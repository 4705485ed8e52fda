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

# The 256- / 512-point tiers of the pruned fast field are used only when they
# carry enough work (csrc/afd_capi.cu: AFD_SUB_MIN_EVALS, default 2^30 grid
# evaluations per field: BASELINE c4).  The GPU tests force them on at every
# size so the small cases exercise those kernels too (read when the library
# loads; test_default_tier_choice checks the default in a fresh process).
os.environ.setdefault("AFD_SUB_MIN_EVALS", "0")


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
