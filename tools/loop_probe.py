"""Scratch probe (GPU box): time the device-resident interaction loop (rounds until every true alarm is revealed)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "ftp"
strat = P.Strategy.seqfix() if len(sys.argv) > 2 and sys.argv[2] == "seqfix" else P.Strategy.parall()
maxr = int(sys.argv[3]) if len(sys.argv) > 3 else None
g, alarms = W.graph(name)
opts = P.EngineOptions(1000, 1e-9)
P.interaction_loop(g, alarms, strat, opts, max_rounds=3)
t = time.perf_counter()
tr = P.interaction_loop(g, alarms, strat, opts, max_rounds=maxr)
dt = time.perf_counter() - t
m = P.compute_metrics(tr)
print(f"{name} {strat.kind}: rounds={len(tr.rounds)} total={dt:.3f}s avg/round={1e3*dt/len(tr.rounds):.3f}ms "
      f"rank100T={m.rank_100t} rank90T={m.rank_90t} inversions={m.inversions} auc={m.auc:.4f}", flush=True)
