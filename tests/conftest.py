"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on CPU."""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large inputs (minutes)")


def sha(*arrays) -> str:
    """sha256 over the arrays' bytes (streamed: no copy of multi-GB arrays)."""
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        if a.size == 0:
            continue
        mv = memoryview(a).cast("B")
        for i in range(0, len(mv), 1 << 28):
            h.update(mv[i:i + (1 << 28)])
    return h.hexdigest()


def _load_optional(name):
    path = os.path.join(GOLDEN_DIR, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    with open(path) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_huge():
    """R-MAT s23/s24 records produced by the reference itself (make_golden_huge.py)."""
    return _load_optional("golden_huge.json")


@pytest.fixture(scope="session")
def golden_s26():
    """The headline config, produced by the full oracle run (make_golden_s26.py)."""
    return _load_optional("golden_s26.json")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_big():
    path = os.path.join(GOLDEN_DIR, "golden_big.json")
    if not os.path.exists(path):
        pytest.skip("golden_big.json not generated")
    with open(path) as fh:
        return json.load(fh)
