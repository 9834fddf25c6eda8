"""Scratch probe (GPU box): where the single-graph e2e time goes (fresh layout per run)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W, _native
w = W.build("C4-PARALL"); g = w.graph
sched = w.strategy.compile(g); arrs = sched.arrays(g)
opts = P.EngineOptions(1000, 1e-9)
for rep in range(8):
    P.engine.clear_device_cache()
    t0 = time.perf_counter(); ga = _native.GraphArrays(g)
    t1 = time.perf_counter(); dg = P.engine.device_graph(g)
    t2 = time.perf_counter(); pl = dg.plan(sched, g)
    t3 = time.perf_counter(); r = pl.run(opts, g)
    t4 = time.perf_counter()
    print(f"arrays {1e3*(t1-t0):.1f} graph_create {1e3*(t2-t1):.1f} plan {1e3*(t3-t2):.1f} run {1e3*(t4-t3):.1f} ms (device {r.device_ms:.2f})", flush=True)
