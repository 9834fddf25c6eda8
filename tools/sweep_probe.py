"""Scratch probe (GPU box): time the C5 multi-evidence sweep (ftp, N sets) on one GPU."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g, alarms = W.graph("ftp")
sets = [W.evidence_set(alarms, j) for j in range(n)]
sel = np.sort(np.asarray(alarms.alarms))
opts = P.EngineOptions(1000, 1e-9)
for r in range(reps):
    t = time.perf_counter()
    res = P.run_many(g, sets, P.Strategy.parall(), opts, marginals=False, deltas=False, select=sel,
                     topk=100, capacity=cap)
    wall = time.perf_counter() - t
    upd = res.total_updates()
    print(f"n={n} passes={res.passes} it[min,max]=[{res.iterations.min()},{res.iterations.max()}] "
          f"kernel_ms={res.kernel_ms:.2f} device_ms={res.device_ms:.2f} wall_ms={wall*1e3:.1f} "
          f"upd/s(kernel)={upd/(res.kernel_ms*1e-3):.3e} errors={sum(e is not None for e in res.errors)}",
          flush=True)
