"""The C-ABI library: loads without a GPU and exports every declared symbol."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2509_22337_b200 import _native

HEADER = os.path.join(ROOT, "include", "hornbp_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hbp_[a-z_]+)\s*\(", text)))


def test_library_exists_and_loads():
    assert os.path.exists(_native.LIB_PATH)
    lib = _native.lib()
    assert b"sm_100a" in lib.hbp_version()


def test_every_header_symbol_is_exported():
    raw = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(raw, s)]
    assert declared_symbols(), "header parse found no symbols"
    assert missing == []


def test_binding_covers_header():
    assert set(declared_symbols()) <= set(_native.EXPORTED)


def test_toposort_layers_and_cycle():
    order = _native.toposort(5, np.array([3, 1]), np.array([0, 0]))
    # layer 0: {1, 2, 3, 4} ascending, then 0
    assert order.tolist() == [1, 2, 3, 4, 0]
    with pytest.raises(_native.NativeError) as err:
        _native.toposort(3, np.array([0, 1]), np.array([1, 0]))
    assert err.value.status == _native.HBP_ECYCLE
    assert err.value.cycle_edge == 0


def test_device_calls_fail_loudly_without_gpu():
    """No CPU fallback: without a usable device the engine raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2509_22337_b200 as P
    from builders import example_graph

    g = example_graph()
    with pytest.raises(RuntimeError):
        P.run(g, P.Strategy.parall().compile(g))
