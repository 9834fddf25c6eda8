import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W, EngineOptions
for name, n in [("weblech", 300), ("hedc", 160), ("weblech", 1000), ("hedc", 640)]:
    g, alarms = W.graph(name)
    rng = np.random.default_rng(2025)
    ids = np.asarray(alarms.alarms); labels = np.asarray(alarms.labels)
    sets = []
    for j in range(n):
        k = int(rng.integers(0, min(10, len(ids)) + 1))
        pick = rng.choice(len(ids), k, replace=False)
        sets.append(list(zip(ids[pick].tolist(), labels[pick].tolist())))
    r = P.run_many(g, sets, None, EngineOptions(1000, 1e-9))
    print(name, n, "compactions", r.compactions, "iters", r.iterations.min(), r.iterations.max())
