"""Scratch probe (GPU box): C5 sweep in fp32 mode vs fp64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
g, alarms = W.graph("ftp")
sets = [W.evidence_set(alarms, j) for j in range(1024)]
sel = np.sort(np.asarray(alarms.alarms))
for prec in ("fp64", "fp32", "fp64", "fp32"):
    r = P.run_many(g, sets, None, P.EngineOptions(1000, 1e-9, precision=prec), marginals=False,
                   deltas=False, select=sel, topk=100)
    print(prec, f"kernel_ms={r.kernel_ms:.2f} it[min,mean,max]=[{r.iterations.min()},{r.iterations.mean():.2f},{r.iterations.max()}] "
          f"upd/s={r.total_updates() / (r.kernel_ms * 1e-3):.3e} compactions={r.compactions}", flush=True)
    if prec == "fp64":
        p64, k64 = r.p1_select.copy(), r.ranked.copy()
    else:
        print("   max |P1 fp32 - fp64| over alarms:", float(np.abs(r.p1_select - p64).max()),
              " top-10 identical sets:", int((r.ranked[:, :10] == k64[:, :10]).all(1).sum()), "/ 1024")
