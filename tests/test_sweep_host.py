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


def test_sweep_algorithmic_bytes_formula():
    """bench.sweep_set_bytes restates DESIGN.md's per-set byte count; check it
    against a direct count of what the staged kernel moves for tiny graphs."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location(
        "bench", os.path.join(os.path.dirname(os.path.dirname(__file__)), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    g, _ = W.graph("weblech")
    V, F, E = g.num_variables, g.num_factors, g.num_edges
    deg = np.diff(np.asarray(g.rowptr))
    T = int(deg[deg > 1].sum())
    for n, max_it in ((1, 1000), (5, 1000), (7, 7)):
        # factor side: iteration 1 writes all E, later ones read + write T;
        # variable side n times: read E ftov + V evidence bytes, write V P0,
        # read V P0 after the first, write T vtof unless the run hit max_iterations
        fac = 16 * E + (n - 1) * 32 * T
        var = n * (16 * E + V) + n * 8 * V + (n - 1) * 8 * V + (n - (n == max_it)) * 16 * T
        idx = n * (4 * (V + 1) + 4 * E + 4 * (F + 1) + 4 * E + 16 * F) / 32.0
        got = float(bench.sweep_set_bytes(g, np.array([n]), max_it)[0])
        assert got == fac + var + idx


def test_evidence_csr_equals_the_list_form():
    """EvidenceCSR (run_many's bulk input) is exactly the conversion of the
    same sets in list / array-pair form; bad CSR and out-of-range variables
    raise like the list form."""
    import numpy as np
    import pytest
    from paper_2509_22337_b200 import EvidenceCSR, workloads as W
    from paper_2509_22337_b200.graph import GraphError
    from paper_2509_22337_b200.sweep import _normalise_sets
    g, alarms = W.graph("weblech")
    sets = [W.evidence_set(alarms, j, size=5) for j in range(7)] + [[(3, True), (4, 0)], []]
    want = _normalise_sets(g, sets)
    csr = EvidenceCSR.from_sets(g, sets)
    got = _normalise_sets(g, csr)
    for a, b in zip(want, got):
        assert np.array_equal(a, b)
    assert len(csr) == len(sets)
    with pytest.raises(ValueError):
        EvidenceCSR([0, 3], [1, 2], [1, 0])
    with pytest.raises(GraphError):
        _normalise_sets(g, EvidenceCSR([0, 1], [g.num_variables], [1]))


def test_evidence_csr_slicing_and_indexing():
    g, _ = W.graph("weblech")
    sets = [[(1, True), (2, False)], [], [(3, False)], [(4, True), (5, True), (6, False)]]
    csr = P.EvidenceCSR.from_sets(g, sets)
    assert [csr[j] for j in range(len(csr))] == sets
    assert csr[-1] == sets[-1]
    part = csr[1:4]
    assert isinstance(part, P.EvidenceCSR) and len(part) == 3
    assert [part[j] for j in range(3)] == sets[1:4]
    assert part.offsets[0] == 0
    assert len(csr[3:1]) == 0
    with pytest.raises(IndexError):
        csr[4]


def test_alarms_to_text_matches_reference_format():
    from paper_2509_22337_b200.ranking import AlarmSet, alarms_to_text

    assert alarms_to_text(AlarmSet((), ())) == "\n"
    assert alarms_to_text(AlarmSet((3, 7), (True, False))) == "alarm 3 1\nalarm 7 0\n"
