"""Shared fixtures; registers the `gpu` marker (tests that need a B200)."""

from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")

# The running example of the reference test-suite (reference tests/conftest.py:12-18):
# a 4-clique {0,1,2,3} sharing vertex 0 with a triangle {0,4,5}.
K4_TRIANGLE_EDGES = [
    (0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3),
    (0, 4), (0, 5), (4, 5),
]
K4_TRIANGLE_CLIQUES = {(0, 1, 2, 3), (0, 4, 5)}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


_golden_cache = None


def golden_cases():
    global _golden_cache
    if _golden_cache is None:
        with open(GOLDEN) as fh:
            _golden_cache = json.load(fh)["cases"]
    return _golden_cache


@pytest.fixture(scope="session")
def golden():
    return golden_cases()
