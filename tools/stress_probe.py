"""Scratch probe (GPU box): randomized parity stress beyond the test suite --
random graphs (up to a few hundred nodes), PARALL / canonical SEQFIX /
random-order SEQFIX / random CUSTOM posets, random options, single runs and
evidence sweeps, every result bitwise against the C oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from builders import random_graph, random_poset
from oracle import orc
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import EngineOptions, Strategy, clamp_evidence

n_graphs = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
t0 = time.time()
checked = 0
ncompact = 0
for trial in range(n_graphs):
    big = trial % 4 == 0
    g = random_graph(rng, max_vars=400 if big else 30, max_factors=400 if big else 30,
                     max_body=int(rng.integers(1, 9)), or_prob=float(rng.uniform(0.2, 0.7)))
    opts = EngineOptions(max_iterations=int(rng.integers(1, 60)),
                         tolerance=float(rng.choice([0.0, 1e-12, 1e-9, 1e-6])),
                         normalize_messages=bool(rng.random() < 0.85))
    kind = trial % 4
    if kind == 0:
        strat = Strategy.parall()
    elif kind == 1:
        strat = Strategy.seqfix()
    elif kind == 2:
        edges = g.edge_list()
        strat = Strategy.seqfix([edges[int(i)] for i in rng.permutation(len(edges))])
    else:
        strat = Strategy.custom(list(random_poset(rng, g, float(rng.uniform(0.1, 0.9))).pairs))
    try:
        sched = strat.compile(g)
    except Exception:
        continue  # e.g. a cyclic random poset: the compiler's error path
    try:
        res = P.run(g, sched, opts)
        err = None
    except P.UnderflowError as e:
        res, err = None, e
    o = orc.run(g, sched.arrays(g), opts.max_iterations, opts.tolerance, opts.normalize_messages,
                threads=4)
    if o["underflow"] is not None:
        assert err is not None, trial
    else:
        assert err is None, (trial, err)
        assert res.iterations == o["iterations"], trial
        assert res.marginals.tobytes() == o["marginals"].tobytes(), trial
        assert np.asarray(res.deltas).tobytes() == o["deltas"].tobytes(), trial
    checked += 1
    if kind == 0 and opts.normalize_messages:
        # evidence sweep of the same graph against clamp_evidence + PARALL
        V = g.num_variables
        sets = []
        for _ in range(int(rng.integers(200, 600)) if trial % 8 == 0 else int(rng.integers(1, 80))):
            k = int(rng.integers(0, min(6, V) + 1))
            sets.append([(int(v), bool(rng.integers(0, 2))) for v in rng.choice(V, k, replace=False)])
        sw = P.run_many(g, sets, None, opts)
        ncompact += sw.compactions
        for j, pairs in enumerate(sets):
            cur = g
            for v, b in pairs:
                cur = clamp_evidence(cur, v, b)
            sc = Strategy.parall().compile(cur)
            oo = orc.run(cur, sc.arrays(cur), opts.max_iterations, opts.tolerance, True, threads=4)
            if oo["underflow"] is not None:
                assert sw.errors[j] is not None, (trial, j)
                continue
            assert sw.errors[j] is None, (trial, j)
            assert sw.iterations[j] == oo["iterations"], (trial, j)
            assert sw.marginals[j].tobytes() == oo["marginals"].tobytes(), (trial, j)
print(f"stress ok: {checked} runs checked ({ncompact} sweep compactions) in {time.time() - t0:.0f} s")
