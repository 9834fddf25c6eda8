"""Scratch probe (GPU box): the bench's sweep step (run_many with device
outputs) timed with CUDA events, against the sweep kernel's own time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
g, alarms = W.graph("ftp")
sets = [W.evidence_set(alarms, j) for j in range(1024)]
sel = np.sort(np.asarray(alarms.alarms, dtype=np.int32))
opts = P.EngineOptions(1000, 1e-9)
dev = torch.device("cuda", 0)
p1 = torch.empty((1024, len(sel)), dtype=torch.float64, device=dev)
rk = torch.empty((1024, 100), dtype=torch.int32, device=dev)
dg = P.engine.device_graph(g)
dg.set_stream(torch.cuda.current_stream(dev))
def step():
    return P.run_many(g, sets, None, opts, marginals=False, deltas=False, select=sel, topk=100,
                      device_out={"p1_select": p1, "ranked": rk})
for _ in range(3):
    step()
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t = time.perf_counter(); e0.record()
    r = step()
    e1.record(); torch.cuda.synchronize()
    print(f"step {e0.elapsed_time(e1):.2f} ms (wall {1e3*(time.perf_counter()-t):.2f}) kernel {r.kernel_ms:.2f} device {r.device_ms:.2f}", flush=True)
import cProfile, pstats, io
pr = cProfile.Profile()
pr.enable(); r = step(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(12); print(s.getvalue()[:3000])
print("c-side wall_ms", r.wall_ms if hasattr(r, "wall_ms") else None)
