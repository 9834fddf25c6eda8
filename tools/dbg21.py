import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from builders import random_graph, random_poset
from oracle import orc
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import EngineOptions, Strategy
rng = np.random.default_rng(2024)
for trial in range(120):
    g = random_graph(rng, max_vars=14, max_factors=14, max_body=4, or_prob=0.5)
    kind = trial % 4
    if kind == 0: sched = Strategy.parall().compile(g)
    elif kind == 1: sched = P.compile_schedule(g, random_poset(rng, g))
    elif kind == 2: sched = Strategy.seqfix(g.edges_at(rng.permutation(g.num_edges))).compile(g)
    else: sched = Strategy.seqfix().compile(g)
    opts = EngineOptions(max_iterations=int(rng.integers(1, 40)), tolerance=float(rng.choice([0.0, 1e-9, 1e-5])), normalize_messages=bool(trial % 5 != 2))
    if trial != 21: continue
    s_off, s_e, t_off, t_e = sched.arrays(g)
    print("trial", trial, "kind", kind, "V", g.num_variables, "F", g.num_factors, "E", g.num_edges, "batches", len(s_off)-1, "opts", opts)
    print("s_off", list(s_off), "t_off", list(t_off))
    o = orc.run(g, sched.arrays(g), opts.max_iterations, opts.tolerance, opts.normalize_messages)
    print("oracle it", o["iterations"], o["underflow"])
    for env in ({}, {"HBP_FUSE": "0"}, {"HBP_SMALL": "0"}):
        for k in ("HBP_FUSE", "HBP_SMALL"): os.environ.pop(k, None)
        os.environ.update(env); P.engine.clear_device_cache()
        try:
            r = P.run(g, sched, opts); print(env, "it", r.iterations, "bits equal", r.marginals.tobytes() == o["marginals"].tobytes())
        except Exception as e: print(env, "exc", e)
    for mi in (1, 2, 3):
        for k in ("HBP_FUSE", "HBP_SMALL"): os.environ.pop(k, None)
        P.engine.clear_device_cache()
        o = orc.run(g, sched.arrays(g), mi, 0.0, True)
        r = P.run(g, sched, EngineOptions(mi, 0.0))
        print("max_it", mi, "equal", r.marginals.tobytes() == o["marginals"].tobytes(), r.marginals[:3, 1], o["marginals"][:3, 1])
    os.environ["HBP_GRID"] = "2"; P.engine.clear_device_cache()
    r = P.run(g, sched, opts); print("grid2 it", r.iterations)
