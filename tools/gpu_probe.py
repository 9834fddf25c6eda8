"""Scratch probe: CUDA path vs C oracle on the BASELINE configs (+ timings)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W
from oracle import orc

names = sys.argv[1:] or ["C1", "C2", "C2-canonical", "C4-PARALL", "C4-SEQFIX", "C3"]
for name in names:
    t = time.time()
    w = W.build(name)
    sched = w.strategy.compile(w.graph)
    tb = time.time() - t
    opts = P.EngineOptions(max_iterations=w.max_iterations, tolerance=w.tolerance)
    o = orc.run(w.graph, sched.arrays(w.graph), w.max_iterations, w.tolerance, threads=8)
    r = P.run(w.graph, sched, opts)  # includes layout + plan build
    times = []
    for _ in range(5):
        t = time.time(); r = P.run(w.graph, sched, opts); times.append(time.time() - t)
    same = r.marginals.tobytes() == o["marginals"].tobytes()
    dsame = list(r.deltas) == list(o["deltas"])
    maxdiff = float(np.max(np.abs(r.marginals - o["marginals"])))
    print(f"{name}: k={sched.num_batches} it gpu={r.iterations} orc={o['iterations']} conv={r.converged} "
          f"bitwise={same} deltas={dsame} maxdiff={maxdiff:.3e} device_ms={r.device_ms:.3f} "
          f"wall_ms={min(times)*1e3:.3f} upd/iter={r.updates_per_iteration} build_s={tb:.2f}", flush=True)
    if not same:
        bad = np.flatnonzero(np.any(r.marginals != o["marginals"], axis=1))
        print("   first bad vars", bad[:10], r.marginals[bad[:3]], o["marginals"][bad[:3]])
        print("   gpu deltas", r.deltas[:5], "orc", list(o["deltas"][:5]))
