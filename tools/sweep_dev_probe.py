"""Probe (GPU box): the bench's sweep leg (device outputs), with HBP_SWEEP_TIMING=1 set-up /
kernel / output times per pass: python tools/sweep_dev_probe.py [sets] [reps]"""
import os, sys
os.environ.setdefault("HBP_SWEEP_TIMING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g, alarms = W.graph("ftp")
sets = [W.evidence_set(alarms, j) for j in range(n)]
sel = np.sort(np.asarray(alarms.alarms))
p1 = torch.empty((n, len(sel)), dtype=torch.float64, device="cuda")
rk = torch.empty((n, 100), dtype=torch.int32, device="cuda")
opts = P.EngineOptions(1000, 1e-9)
for r in range(reps):
    res = P.run_many(g, sets, P.Strategy.parall(), opts, marginals=False, deltas=False, select=sel,
                     topk=100, device_out={"p1_select": p1, "ranked": rk})
    print(f"kernel_ms={res.kernel_ms:.2f} device_ms={res.device_ms:.2f}", flush=True)
