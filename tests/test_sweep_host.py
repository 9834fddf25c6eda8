"""Host-side logic of the sweep API (no GPU needed)."""

import numpy as np
import pytest

import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import sweep as S
from paper_2509_22337_b200 import workloads as W


def test_normalise_sets_forms():
    g, _ = W.graph("weblech")
    off, var, val = S._normalise_sets(g, [[(1, True), (2, False)], [],
                                          (np.array([3, 4]), np.array([False, True]))])
    assert off.tolist() == [0, 2, 2, 4]
    assert var.tolist() == [1, 2, 3, 4]
    assert val.tolist() == [1, 0, 0, 1]


def test_bad_arguments_raise_before_the_device():
    g, _ = W.graph("weblech")
    with pytest.raises(P.GraphError):
        P.run_many(g, [[(g.num_variables, True)]])
    with pytest.raises(ValueError):
        P.run_many(g, [[]], select=[5, 3])
    with pytest.raises(ValueError):
        P.run_many(g, [[]], topk=3)
    with pytest.raises(ValueError):
        P.run_many(g, [[]], options=P.EngineOptions(record_history=True))
    with pytest.raises(ValueError):
        P.run_many(g, [[]], options=P.EngineOptions(max_iterations=0))
