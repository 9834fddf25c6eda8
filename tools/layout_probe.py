"""Where a fresh graph's device layout time goes (HBP_LAYOUT_TIMING stages),
create and destroy timed separately."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HBP_LAYOUT_TIMING", "1")
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import workloads as W, _native
w = W.build("C4-PARALL"); g = w.graph
sched = w.strategy.compile(g)
opts = P.EngineOptions(1000, 1e-9)
L = _native.lib()
ga = _native.GraphArrays(g)
for rep in range(6):
    h = C.c_void_p()
    t0 = time.perf_counter()
    assert L.hbp_graph_create(C.byref(ga.desc), 0, C.byref(h)) == 0, _native.last_error()
    t1 = time.perf_counter()
    L.hbp_graph_destroy(h)
    t2 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms destroy {1e3*(t2-t1):.2f} ms", file=sys.stderr, flush=True)
os.environ.pop("HBP_LAYOUT_TIMING")
for rep in range(6):
    P.engine.clear_device_cache()
    t0 = time.perf_counter(); r = P.run(g, sched, opts); t1 = time.perf_counter()
    print(f"run() fresh graph {1e3*(t1-t0):.2f} ms (device {r.device_ms:.3f})", file=sys.stderr, flush=True)
