"""The reference-side C-ABI binding (integration/hornbp_gpu.py, shown in
INTEGRATION.md 2): bound with full ctypes signatures, driven from the
reference package's own objects, and checked against hornbp.run itself.

The reference is imported from baseline/_ref (pip --target of
/root/reference/pkg; it travels to the GPU box with the snapshot) -- never
from /root/reference at run time."""

import os
import re
import sys

import numpy as np
import pytest

from conftest import ROOT

REF_SITE = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, os.path.join(ROOT, "integration"))


@pytest.fixture(scope="module")
def R():
    if not os.path.isdir(os.path.join(REF_SITE, "hornbp")):
        pytest.skip("baseline/_ref (the pip-installed reference) not present")
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    import hornbp

    return hornbp


def test_binding_symbols_declared_and_exported():
    import hornbp_gpu

    header = open(os.path.join(ROOT, "include", "hornbp_gpu.h")).read()
    L = hornbp_gpu.lib()
    for name, (res, args) in hornbp_gpu.SIGNATURES.items():
        assert re.search(rf"\b{name}\s*\(", header), name
        fn = getattr(L, name)
        assert fn.argtypes == args and fn.restype == res, name


def mirror(R, g):
    return R.FactorGraph(g.num_variables, [R.Factor(R.FactorKind(f.kind.value), f.head, f.body,
                                                    f.p1, f.p2) for f in g.factors])


@pytest.mark.gpu
def test_binding_bitwise_vs_hornbp_run(R):
    import hornbp_gpu

    g, _ = R.generate(R.SynthSpec(313, 383, 8, 0))  # C1 weblech, the reference's generator
    for strat, opts in ((R.Strategy.parall(), R.EngineOptions(max_iterations=100, tolerance=0.0)),
                        (R.Strategy.seqfix(), R.EngineOptions(max_iterations=1000, tolerance=1e-9)),
                        # explicit-order SEQFIX (TOPO needs a forest; weblech is loopy)
                        (R.Strategy.seqfix(list(reversed(list(g.edges())))),
                         R.EngineOptions(max_iterations=50, tolerance=1e-9, record_history=True))):
        sched = strat.compile(g)
        want = R.run(g, sched, opts)
        got = hornbp_gpu.run(g, sched, opts)
        assert isinstance(got, R.InferenceResult)
        assert got.iterations == want.iterations and got.converged == want.converged
        assert got.marginals.tobytes() == want.marginals.tobytes()
        assert got.deltas == want.deltas
        if want.history is not None:
            assert len(got.history) == len(want.history)
            assert all(a.tobytes() == b.tobytes() for a, b in zip(got.history, want.history))


@pytest.mark.gpu
def test_binding_underflow_and_errors_like_hornbp(R):
    """Same exception type and message as hornbp.run, index included."""
    import hornbp_gpu
    from builders import contradictory_graph

    rng = np.random.default_rng(909)
    raised = 0
    for trial in range(60):
        rg = mirror(R, contradictory_graph(rng))
        sched = (R.Strategy.parall() if trial % 2 else R.Strategy.seqfix()).compile(rg)
        opts = R.EngineOptions(max_iterations=20, tolerance=1e-9)
        try:
            want = R.run(rg, sched, opts)
        except R.UnderflowError as exc:
            with pytest.raises(R.UnderflowError) as ei:
                hornbp_gpu.run(rg, sched, opts)
            assert str(ei.value) == str(exc), trial
            raised += 1
            continue
        got = hornbp_gpu.run(rg, sched, opts)
        assert got.marginals.tobytes() == want.marginals.tobytes(), trial
    assert raised >= 20, raised
    with pytest.raises(ValueError):
        hornbp_gpu.run(rg, sched, R.EngineOptions(max_iterations=0))
