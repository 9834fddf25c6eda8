"""Scratch probe (GPU box): kernel time of the C5 sweep capped at k iterations (tail cost)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
g, alarms = W.graph("ftp")
sets = [W.evidence_set(alarms, j) for j in range(1024)]
for mx in (1000, 23, 24, 26, 28):
    ts = []
    for _ in range(2):
        r = P.run_many(g, sets, options=P.EngineOptions(mx, 1e-9), marginals=False, deltas=False)
        ts.append(r.kernel_ms)
    print(f"max_it={mx}: kernel_ms={min(ts):.2f} set-iterations={int(r.iterations.sum())}", flush=True)
