"""Shared fixtures.  `-m gpu` tests need a B200 (run through gpurun); the
rest run on CPU.  Golden vectors come from the reference package itself
(tests/golden/make_golden.py); /root/reference is never read here."""

from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle check")


def load_json(name: str):
    path = os.path.join(GOLDEN_DIR, name)
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def goldens():
    g = load_json("goldens.json")
    assert g is not None, "tests/golden/goldens.json missing"
    return g


@pytest.fixture(scope="session")
def cfg5_golden():
    g = load_json("cfg5_seed7.json")
    if g is None:
        pytest.skip("cfg5 golden not generated yet")
    return g


def hexrows(rows):
    return [int(r, 16) for r in rows]


# cfg4 histogram checksum (independent numpy
# restatement of the level-3 saved-additions walk)
CFG4_HIST_SHA256 = "8d397da157d31b1e67746a3a522b01cb624e4d54d42a27b6fbd403a6da02252b"


@pytest.fixture(scope="session")
def cfg5_traces():
    g = load_json("cfg5_traces.json")
    if g is None:
        pytest.skip("cfg5 seed traces not generated yet")
    return g


@pytest.fixture(scope="session")
def section6():
    g = load_json("section6_codes.json")
    if g is None:
        pytest.skip("section-6 codes not generated yet")
    return g
