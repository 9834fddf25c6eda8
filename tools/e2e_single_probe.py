"""Scratch probe (GPU box): the bench's single-graph e2e leg, with and without a sweep created first."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
r = bench.measure_single(torch, "c4", steps=10, warmup=3)
print("fresh process: e2e ms", r["e2e"]["ms_per_step"], "device ms", r["time_to_convergence_ms"], flush=True)
g, alarms = W.graph("ftp")
w = W.build("C4-PARALL")
print("same graph object:", g is w.graph, flush=True)
sets = [W.evidence_set(alarms, j) for j in range(64)]
P.run_many(g, sets, None, P.EngineOptions(1000, 1e-9), marginals=False, deltas=False)
r = bench.measure_single(torch, "c4", steps=10, warmup=3)
print("after a sweep: e2e ms", r["e2e"]["ms_per_step"], flush=True)
sched = w.strategy.compile(w.graph)
opts = P.EngineOptions(1000, 1e-9)
for i in range(5):
    t0 = time.perf_counter(); P.engine.clear_device_cache(); t1 = time.perf_counter()
    res = P.run(w.graph, sched, opts); t2 = time.perf_counter()
    print(f"clear {1e3*(t1-t0):.2f} ms run {1e3*(t2-t1):.2f} ms", flush=True)
