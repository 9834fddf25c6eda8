"""Shared test configuration.

Markers:
  gpu  -- needs a CUDA device (run on the B200 box: pytest -m gpu)

Tests never read /root/reference at run time on the GPU box; in the
development container, tests marked ``needs_ref`` additionally compare
against the reference package when it is present.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/pkg/src"
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200)")
    config.addinivalue_line("markers", "needs_ref: requires /root/reference (dev container only)")


def pytest_collection_modifyitems(config, items):
    have_ref = os.path.isdir(REF_SRC)
    for item in items:
        if "needs_ref" in item.keywords and not have_ref:
            item.add_marker(pytest.mark.skip(reason="reference package not present"))


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def hornbp_ref():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import hornbp

    return hornbp


def sha(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sched_sha(arrs) -> str:
    import hashlib

    return hashlib.sha256(b"".join(np.ascontiguousarray(a).tobytes() for a in arrs)).hexdigest()
