"""Shared test setup.

Markers: ``gpu`` -- needs a CUDA device (sm_100a) and libpk.so; everything
else runs on the CPU (the driver runs ``-m "not gpu"`` without a GPU).
Only tests/ may import ``oracle`` (test infrastructure).
"""

import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and libpk.so")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "interp_vectors.json")) as fh:
        return json.load(fh)["vectors"]


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1801_04348_b200 import _lib

    _lib.load()
    return torch
