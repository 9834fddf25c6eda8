"""Scratch probe (GPU box): where the time of one device interaction round goes (ftp)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
g, alarms = W.graph(sys.argv[1] if len(sys.argv) > 1 else "ftp")
opts = P.EngineOptions(1000, 1e-9)
sched = P.Strategy.parall().compile(g)
dg = P.engine.device_graph(g)
plan = dg.plan(sched, g)
sel = np.unique(np.asarray(alarms.alarms, dtype=np.int32))
ev_v, ev_l = [], []
T = {"ev": 0.0, "run": 0.0, "rank": 0.0}
its = []
for r in range(400):
    t0 = time.perf_counter(); dg.set_evidence(ev_v, ev_l)
    t1 = time.perf_counter(); res = plan.run_device(opts, g)
    t2 = time.perf_counter(); top, p1 = dg.rank(sel, 1)
    t3 = time.perf_counter()
    if r >= 10:
        T["ev"] += t1 - t0; T["run"] += t2 - t1; T["rank"] += t3 - t2
    its.append(res.iterations)
    ev_v.append(int(top[0])); ev_l.append(int(alarms.label_of(int(top[0]))))
n = 390
print({k: f"{1e3 * v / n:.3f} ms" for k, v in T.items()}, "iterations first/last", its[:3], its[-3:],
      "device_ms last", res.device_ms)
