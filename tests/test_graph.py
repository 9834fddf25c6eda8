"""Graph model: validation, FASTFG, DAG conversion, clamping."""

import pytest

from builders import example_graph
from paper_2509_22337_b200 import (DagNode, EdgeId, Factor, FactorGraph, FactorKind, FormatError,
                                   GraphError, clamp_evidence, from_bayesian_dag, parse_dag,
                                   parse_fastfg)
from paper_2509_22337_b200 import workloads as W


def test_parse_and_roundtrip():
    text = "FASTFG 1\nvars 3\nfactor AND 0.999 0.0 head=2 body=0,1\nfactor AND 0.5 0.5 head=0 body=\nfactor AND 0.5 0.5 head=1 body=\n"
    g = parse_fastfg(text)
    assert (g.num_variables, g.num_factors, g.num_edges) == (3, 3, 5)
    f = g.factors[0]
    assert f.kind is FactorKind.AND and f.head == 2 and f.body == (0, 1)
    assert parse_fastfg(g.to_fastfg()).to_fastfg() == g.to_fastfg()


def test_comments_blank_lines():
    g = parse_fastfg("# x\nFASTFG 1\n\nvars 2 # two\nfactor OR 1.0 0.0 head=0 body=1\nfactor AND 0.5 0.5 head=1 body=\n")
    assert g.factors[0].kind is FactorKind.OR


@pytest.mark.parametrize("line,frag", [
    ("factor NAND 0.9 0.0 head=0 body=1", "kind"),
    ("factor AND 1.5 0.0 head=0 body=1", "probability"),
    ("factor AND 0.9 0.0 head=0 body=1,1", "duplicate"),
    ("factor AND 0.9 0.0 head=0 body=0", "head"),
    ("factor AND 0.9 0.0 head=0", "expected"),
    ("factor AND 0.9 0.0 head=5 body=0", "out of range"),
])
def test_format_errors_carry_line(line, frag):
    with pytest.raises(FormatError) as err:
        parse_fastfg(f"FASTFG 1\nvars 2\n{line}\n")
    assert err.value.line == 3 and frag in str(err.value)


def test_missing_header_and_vars():
    with pytest.raises(FormatError):
        parse_fastfg("vars 2\n")
    with pytest.raises(FormatError):
        parse_fastfg("FASTFG 1\n")


@pytest.mark.parametrize("factors,frag", [
    ([Factor(FactorKind.AND, 0, (0,), 0.5, 0.1)], "head variable repeated"),
    ([Factor(FactorKind.AND, 1, (0, 0), 0.5, 0.1)], "duplicate body"),
    ([Factor(FactorKind.AND, 0, (), 0.5, 0.4), Factor(FactorKind.AND, 1, (), .5, .5)], "p1 == p2"),
    ([Factor(FactorKind.OR, 0, (), 0.5, 0.5), Factor(FactorKind.AND, 1, (), .5, .5)], "OR factor"),
    ([Factor(FactorKind.AND, 0, (), 1.5, 1.5), Factor(FactorKind.AND, 1, (), .5, .5)], "outside"),
    ([Factor(FactorKind.AND, 0, (), 0.5, 0.5)], "appears in no factor"),
    ([Factor(FactorKind.AND, 0, (7,), 0.5, 0.1)], "out of range"),
])
def test_validation_messages(factors, frag):
    with pytest.raises(GraphError, match=frag):
        FactorGraph(2, factors)


def test_edges_adjacency_and_indices():
    g = example_graph()
    assert g.edge_list() == [EdgeId(0, 0), EdgeId(1, 0), EdgeId(2, 0), EdgeId(2, 1), EdgeId(2, 2)]
    assert g.adjacency == (((0, 0), (2, 1)), ((1, 0), (2, 2)), ((2, 0),))
    assert g.variable_of(EdgeId(2, 2)) == 1
    assert [g.edge_index(e) for e in g.edges()] == list(range(5))
    with pytest.raises(GraphError):
        g.check_edge(EdgeId(2, 3))
    with pytest.raises(GraphError):
        g.check_edge(EdgeId(9, 0))


def test_dag_conversion_roles():
    nodes = [DagNode("a", "input", 0.9), DagNode("b", "input"), DagNode("c", "clause", 0.8),
             DagNode("t", "tuple")]
    g = from_bayesian_dag(nodes, [("a", "c"), ("b", "c"), ("c", "t")])
    assert g.names == ("a", "b", "c", "t")
    f = g.factors
    assert (f[0].kind, f[0].p1, f[0].p2, f[0].body) == (FactorKind.AND, 0.9, 0.9, ())
    assert f[1].p1 == 0.999
    assert (f[2].kind, f[2].head, f[2].body, f[2].p1, f[2].p2) == (FactorKind.AND, 2, (0, 1), 0.8, 0.0)
    assert (f[3].kind, f[3].body, f[3].p1, f[3].p2) == (FactorKind.OR, (2,), 1.0, 0.0)


@pytest.mark.parametrize("nodes,edges,frag", [
    ([DagNode("a", "input"), DagNode("a", "input")], [], "declared twice"),
    ([DagNode("a", "weird")], [], "unknown role"),
    ([DagNode("t", "tuple", 0.5)], [], "no probability"),
    ([DagNode("t", "tuple")], [], "no deriving clause"),
    ([DagNode("c", "clause")], [], "no premises"),
    ([DagNode("a", "input")], [("a", "z")], "unknown node"),
    ([DagNode("x", "clause"), DagNode("y", "clause")], [("x", "y"), ("y", "x")], "cycle"),
])
def test_dag_errors(nodes, edges, frag):
    with pytest.raises(GraphError, match=frag):
        from_bayesian_dag(nodes, edges)


def test_parse_dag():
    g = parse_dag("node a input p=0.7\nnode c clause\nnode t tuple\nedge a c\nedge c t\n")
    assert g.num_variables == 3 and g.factors[1].p1 == 0.999
    with pytest.raises(FormatError):
        parse_dag("node a input q=1\n")
    with pytest.raises(FormatError):
        parse_dag("bogus a\n")


def test_clamp_appends_and_keeps_edges():
    g = example_graph()
    c = clamp_evidence(g, 1, True)
    assert c.num_factors == 4 and g.num_factors == 3
    pin = c.factors[-1]
    assert pin.arity == 0 and pin.p1 == pin.p2 == 1.0
    assert clamp_evidence(g, 1, False).factors[-1].p1 == 0.0
    for e in g.edges():
        assert c.edge_index(e) == g.edge_index(e)
    with pytest.raises(GraphError):
        clamp_evidence(g, 7, True)


def test_factor_objects_lazy_equal_eager():
    g, _ = W.graph("weblech")
    eager = FactorGraph(g.num_variables, g.factors, g.names)
    assert eager.to_fastfg() == g.to_fastfg()
    assert (eager.rowptr == g.rowptr).all() and (eager.vars == g.vars).all()
