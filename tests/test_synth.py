"""Generator parity: the BASELINE graphs are byte-identical to the reference's."""

import hashlib

import numpy as np
import pytest

from conftest import sha
from paper_2509_22337_b200 import SynthError, SynthSpec, generate
from paper_2509_22337_b200 import workloads as W


@pytest.mark.parametrize("name", ["weblech", "hedc", "avrora", "ftp"])
def test_baseline_graph_checksums(name, golden):
    g, alarms = W.graph(name)
    want = golden["graphs"][name]
    assert (g.num_variables, g.num_edges, g.num_factors) == (want["V"], want["E"], want["F"])
    assert hashlib.sha256(g.to_fastfg().encode()).hexdigest() == want["fastfg_sha"]
    assert want["fastfg_sha"].startswith(W.FASTFG_SHA[name])
    assert sha(np.asarray(alarms.alarms, dtype=np.int64)) == want["alarms_sha"]
    assert sha(np.asarray(alarms.labels, dtype=np.int8)) == want["labels_sha"]


def test_weblech_size_matches_paper_table():
    g, _ = generate(SynthSpec(313, 383, 8, 0))
    assert g.num_variables == 313 + 383 == 696


def test_deterministic():
    a = generate(SynthSpec(60, 80, 4, 9))
    b = generate(SynthSpec(60, 80, 4, 9))
    assert a[0].to_fastfg() == b[0].to_fastfg() and a[1] == b[1]


def test_tree_mode_is_a_forest():
    from paper_2509_22337_b200 import Strategy

    g, _ = generate(SynthSpec(30, 20, 8, 3, tree_only=True))
    Strategy.topo().compile(g)  # raises on a cycle


@pytest.mark.parametrize("spec,msg", [
    (SynthSpec(0, 0), "at least one tuple"),
    (SynthSpec(0, 3), "zero tuples"),
    (SynthSpec(1, 1), "two tuples"),
    (SynthSpec(5, -1), "nonnegative"),
    (SynthSpec(5, 2, max_premises=0), "max_premises"),
    (SynthSpec(3, 5, tree_only=True), "tree mode"),
    (SynthSpec(5, 2, clause_prob=0.0), "clause_prob"),
])
def test_infeasible_specs(spec, msg):
    with pytest.raises(SynthError, match=msg):
        generate(spec)


@pytest.mark.needs_ref
@pytest.mark.parametrize("spec", [(10, 12, 3, 1), (40, 90, 8, 5), (200, 150, 2, 7),
                                  (25, 20, 8, 2, True), (2, 1, 8, 0), (7, 0, 8, 4)])
def test_matches_reference_generator(spec, hornbp_ref):
    mine = generate(SynthSpec(*spec))
    ref = hornbp_ref.generate(hornbp_ref.SynthSpec(*spec))
    assert mine[0].to_fastfg() == ref[0].to_fastfg()
    assert mine[0].names == ref[0].names
    assert mine[1].alarms == ref[1].alarms and mine[1].labels == ref[1].labels
