import ctypes as C, os, sys, json
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W, _native
gold = json.load(open('/root/repo/tests/golden/golden.json'))["runs"]["C1"]
w = W.build("C1"); g = w.graph
sched = w.strategy.compile(g)
res = P.run(g, sched, P.EngineOptions(max_iterations=100, tolerance=0.0))
ok = [float(d).hex() for d in res.deltas] == gold["deltas"]
plan = P.engine.device_graph(g).plan(sched, g)
nph, grid, thr = C.c_int32(), C.c_int32(), C.c_int32()
_native.lib().hbp_debug_plan_info(plan.handle, C.byref(nph), C.byref(grid), C.byref(thr))
print("HBP_DYN", os.environ.get("HBP_DYN"), "ok", ok, "nphases", nph.value, "grid", grid.value, "threads", thr.value, "V", g.num_variables, "F", g.num_factors, "E", g.num_edges)
