"""Probe (GPU box): per-iteration device time of a config at a fixed iteration count
(tolerance 0): python tools/iter_probe.py C4-PARALL 50"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
name, iters = sys.argv[1], int(sys.argv[2])
w = W.build(name)
sched = w.strategy.compile(w.graph)
opts = P.EngineOptions(max_iterations=iters, tolerance=0.0)
t = time.time()
while time.time() - t < 1.0:
    r = P.run(w.graph, sched, opts)
ms = [P.run(w.graph, sched, opts).device_ms for _ in range(10)]
print(f"{name} fixed {iters} it: device_ms min={min(ms):.3f} per_iter_us={1e3*min(ms)/iters:.2f}", flush=True)
