"""Probe (GPU box): per-level timeline of a levelled schedule (HBP_TRACE=1),
CTA 0's phase compute time against the level's size."""
import ctypes as C, os, sys, time
os.environ["HBP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import _native, workloads as W
name = sys.argv[1]
w = W.build(name)
sched = w.strategy.compile(w.graph)
opts = P.EngineOptions(max_iterations=w.max_iterations, tolerance=w.tolerance)
t = time.time()
while time.time() - t < 1.0:
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
a = (np.frombuffer(buf, dtype=np.uint64)[:n0].reshape(4, nph, G, 2) >> np.uint64(8)).astype(np.int64)
s_off, s_e, t_off, t_e = sched.arrays(w.graph)
print(f"{name}: device_ms {r.device_ms:.3f} it {r.iterations} phases {nph} fused {v[3].value} grid {G}")
it = 1
st, en = a[it, :, 0, 0], a[it, :, 0, 1]
dur = (en - st) / 1e3
gap = np.r_[0, (st[1:] - en[:-1]) / 1e3]
tot = (en[-1] - st[0]) / 1e3
print(f"iteration 3 CTA0: total {tot:.1f} us, compute sum {dur.sum():.1f}, gaps sum {gap[1:].sum():.1f}")
print("phase 0..3 us:", np.round(dur[:4], 2), "gaps", np.round(gap[:4], 2))
d = dur[2:]
print("small phases: n %d mean %.2f med %.2f p10 %.2f p90 %.2f max %.2f us; mean gap %.2f" % (
    len(d), d.mean(), np.median(d), np.percentile(d, 10), np.percentile(d, 90), d.max(), gap[3:].mean()))
# size of each level (edges in s_b) vs its phase time (fused plans: phase p >= 2 is level p - 1)
if v[3].value == len(s_off) - 2:
    sizes = np.diff(s_off)[1:]
    for lo, hi in ((0, 256), (256, 512), (512, 768), (768, 1024), (1024, 1536), (1536, 4000)):
        m = (sizes >= lo) & (sizes < hi)
        if m.any():
            print(f"  levels with {lo}-{hi} edges: {m.sum():4d}, mean {d[m].mean():.2f} us")

