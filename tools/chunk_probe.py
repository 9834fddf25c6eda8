"""Probe (GPU box, -DHBP_TRACE_CHUNKS build via HBP_LIB_PATH): per-class chunk times of
lbp_parall's two phases in iteration 3. python tools/chunk_probe.py C4-PARALL"""
import ctypes as C, os, sys, time
os.environ["HBP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import _native, workloads as W
w = W.build(sys.argv[1] if len(sys.argv) > 1 else "C4-PARALL")
sched = w.strategy.compile(w.graph)
opts = P.EngineOptions(max_iterations=w.max_iterations, tolerance=w.tolerance)
for _ in range(3):
    r = P.run(w.graph, sched, opts)
plan = P.engine.device_graph(w.graph).plan(sched, w.graph)
lib = _native.lib()
lib.hbp_debug_trace.restype = C.c_int64
lib.hbp_debug_trace.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int64]
v = [C.c_int32() for _ in range(4)]
lib.hbp_debug_plan_info(plan.handle, *[C.byref(x) for x in v])
nph, G = v[0].value, v[1].value
n0 = 4 * nph * G * 2
n = n0 + 2 * 16384
buf = (C.c_ulonglong * n)()
lib.hbp_debug_trace(plan.handle, buf, n)
ch = np.frombuffer(buf, dtype=np.uint64)[n0:].reshape(2, 16384)
for ph in range(2):
    x = ch[ph]
    x = x[x > 0]
    ns = (x & np.uint64((1 << 48) - 1)).astype(np.int64)
    cls = (x >> np.uint64(48)).astype(np.int64)
    print(f"phase {ph}: {len(x)} chunks, total {ns.sum()/1e3:.0f} us-warp")
    for c in np.unique(cls):
        m = cls == c
        print(f"   class {c:2d}: {m.sum():5d} chunks, mean {ns[m].mean():6.0f} ns, p90 {np.percentile(ns[m],90):6.0f}, share {100*ns[m].sum()/ns.sum():5.1f} %")
