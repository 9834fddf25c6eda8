"""Scratch probe (GPU box): per-32-set tile convergence spread of the C5 sweep (straggler overhead)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
g, alarms = W.graph("ftp")
sets = [W.evidence_set(alarms, j) for j in range(1024)]
r = P.run_many(g, sets, marginals=False, deltas=False)
it = r.iterations.astype(int)
print("iterations histogram:", np.bincount(it)[20:])
t = it.reshape(-1, 32)
print("mean set iterations", it.mean(), "mean tile max", t.max(1).mean(), "ratio", t.max(1).mean() / it.mean())
alive_hist = np.zeros(33, int)
for k in range(1, it.max() + 1):
    a = (t >= k).sum(1)
    for x in a[a > 0]:
        alive_hist[x] += 1
print("tile-iterations by alive lanes (1..32):", alive_hist[1:].tolist())
