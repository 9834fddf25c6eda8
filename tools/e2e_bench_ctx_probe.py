"""Scratch probe (GPU box): single-graph e2e after the bench's 1,024-set sweeps (the bench's own order)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W, _native
g, alarms = W.graph("ftp")
sets = [W.evidence_set(alarms, j) for j in range(1024)]
P.run_many(g, sets, None, P.EngineOptions(1000, 1e-9), marginals=False, deltas=False)
P.run_many(g, sets, None, P.EngineOptions(1000, 1e-9, precision="fp32"), marginals=False, deltas=False)
flush = torch.empty(256 << 20 >> 2, dtype=torch.float32, device="cuda")
w = W.build("C4-PARALL")
sched = w.strategy.compile(w.graph)
opts = P.EngineOptions(1000, 1e-9)
L = _native.lib()
for i in range(12):
    t0 = time.perf_counter(); P.engine.clear_device_cache(); t1 = time.perf_counter()
    dg = P.engine.device_graph(w.graph); t2 = time.perf_counter()
    pl = dg.plan(sched, w.graph); t3 = time.perf_counter()
    r = pl.run(opts, w.graph); t4 = time.perf_counter()
    del pl, dg
    print(f"clear {1e3*(t1-t0):.2f} create {1e3*(t2-t1):.2f} plan {1e3*(t3-t2):.2f} run {1e3*(t4-t3):.2f} ms", flush=True)
