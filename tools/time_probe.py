"""Scratch probe (GPU box): warm the GPU, then time repeated runs of one config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = W.build(name)
sched = w.strategy.compile(w.graph)
opts = P.EngineOptions(max_iterations=w.max_iterations, tolerance=w.tolerance)
t = time.time()
while time.time() - t < 2.0:
    r = P.run(w.graph, sched, opts)
ms = []
for _ in range(reps):
    r = P.run(w.graph, sched, opts)
    ms.append(r.device_ms)
print(f"{name} it={r.iterations} device_ms min={min(ms):.3f} med={np.median(ms):.3f} per_iter_us={1e3*min(ms)/r.iterations:.2f}", flush=True)
