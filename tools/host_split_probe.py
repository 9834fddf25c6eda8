"""Scratch probe (GPU box): run_many's time inside vs outside hbp_sweep_run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W, _native
g, alarms = W.graph("ftp")
sets = P.EvidenceCSR.from_sets(g, [W.evidence_set(alarms, j) for j in range(1024)])
sel = np.sort(np.asarray(alarms.alarms, dtype=np.int32))
opts = P.EngineOptions(1000, 1e-9)
dev = torch.device("cuda", 0)
p1 = torch.empty((1024, len(sel)), dtype=torch.float64, device=dev)
rk = torch.empty((1024, 100), dtype=torch.int32, device=dev)
L = _native.lib()
orig = L.hbp_sweep_run
T = []
def timed(*a):
    t = time.perf_counter(); st = orig(*a); T.append(time.perf_counter() - t); return st
L.hbp_sweep_run = timed
for i in range(6):
    t = time.perf_counter()
    r = P.run_many(g, sets, None, opts, marginals=False, deltas=False, select=sel, topk=100,
                   device_out={"p1_select": p1, "ranked": rk})
    w = time.perf_counter() - t
    if i >= 2:
        print(f"run_many {1e3*w:.2f} ms, hbp_sweep_run {1e3*T[-1]:.2f} ms, kernel {r.kernel_ms:.2f}, device {r.device_ms:.2f}", flush=True)
