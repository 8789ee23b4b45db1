"""Test configuration.

Markers: ``gpu`` tests need a CUDA device (the B200 runs them with
``pytest -m gpu``); everything else runs on the CPU build container.
Tests import the product from the repo root and the oracle from oracle/.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
        return cache[name]

    return load


@pytest.fixture(scope="session")
def golden_variant():
    """zgemm order the fixtures were generated with (tests/golden/META.json)."""
    import json
    return json.loads((GOLDEN / "META.json").read_text())["variant"]


def pytest_collection_modifyitems(config, items):
    have_gpu = False
    try:
        from paper_2310_17739_b200 import _native
        have_gpu = _native.device_count() > 0
    except Exception:
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
