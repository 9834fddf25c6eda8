"""Scratch: per-phase timeline from HBP_TRACE=1 (phase compute vs barrier)."""
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
nph, grid, thr = C.c_int32(), C.c_int32(), C.c_int32()
lib.hbp_debug_plan_info(plan.handle, C.byref(nph), C.byref(grid), C.byref(thr))
nph, G = nph.value, grid.value
n = 4 * nph * G * 2 + (2 * 16384 if nph == 2 else 0)
buf = (C.c_ulonglong * n)()
lib.hbp_debug_trace(plan.handle, buf, n)
allb = np.frombuffer(buf, dtype=np.uint64)
raw = allb[:4 * nph * G * 2].reshape(4, nph, G, 2)
chunk_ns = allb[4 * nph * G * 2:].reshape(2, 16384).astype(np.int64) if nph == 2 else None
a = (raw >> np.uint64(8)).astype(np.int64)
smid = (raw[0, 0, :, 0] & np.uint64(0xff)).astype(np.int64)
print(f"{name}: device_ms {r.device_ms:.3f} iterations {r.iterations} phases {nph} grid {G} threads {thr.value}")
for it in range(min(3, r.iterations - 1)):
    t0 = a[it, 0, :, 0].min()
    tot = []
    for p in range(min(nph, int(sys.argv[2]) if len(sys.argv) > 2 else 8)):
        st, en = a[it, p, :, 0], a[it, p, :, 1]
        ok = st > 0
        if not ok.any():
            continue
        dur = (en - st)[ok]
        print(f"  it{it+2} ph{p}: start +{(st[ok].min()-t0)/1e3:7.2f}us (spread {(st[ok].max()-st[ok].min())/1e3:5.2f}) "
              f"compute min/med/max {dur.min()/1e3:6.2f}/{np.median(dur)/1e3:6.2f}/{dur.max()/1e3:6.2f}us  end max +{(en[ok].max()-t0)/1e3:7.2f}")
    if nph > 8:
        # summary over all phases of this iteration
        starts = a[it, :, 0, 0]; ends = a[it, :, 0, 1]
        d = (ends - starts)[starts > 0]
        gaps = starts[1:] - ends[:-1]
        print(f"  it{it+2} CTA0: phases {len(d)} mean compute {d.mean()/1e3:.2f}us mean gap {gaps[gaps>0].mean()/1e3:.2f}us total {(ends.max()-starts[starts>0].min())/1e3:.1f}us")

# per-CTA phase-0 durations: stable across iterations (static imbalance) or noise?
its = min(4, r.iterations - 1)
d0 = np.stack([(a[i, 0, :, 1] - a[i, 0, :, 0]) / 1e3 for i in range(its)])
d1 = np.stack([(a[i, 1, :, 1] - a[i, 1, :, 0]) / 1e3 for i in range(its)]) if nph > 1 else None
print("phase-0 per-CTA duration corr(it2,it3) = %.3f, corr(it3,it4) = %.3f" % (
    np.corrcoef(d0[0], d0[1])[0, 1], np.corrcoef(d0[1], d0[2])[0, 1]))
if d1 is not None:
    print("phase-1 per-CTA duration corr(it2,it3) = %.3f" % np.corrcoef(d1[0], d1[1])[0, 1])
m0 = d0.mean(0)
order = np.argsort(-m0)
print("slowest CTAs (cta, sm, mean us):", [(int(c), int(smid[c]), round(float(m0[c]), 2)) for c in order[:10]])
print("fastest CTAs:", [(int(c), int(smid[c]), round(float(m0[c]), 2)) for c in order[-5:]])
# by SM parity / half (die guess)
for name_, mask in [("sm < 74", smid < 74), ("sm >= 74", smid >= 74), ("even sm", smid % 2 == 0), ("odd sm", smid % 2 == 1)]:
    print(f"  {name_}: mean ph0 {m0[mask].mean():.2f} us" + (f", ph1 {d1.mean(0)[mask].mean():.2f} us" if d1 is not None else ""))

if chunk_ns is not None:
    for ph in range(2):
        cn = chunk_ns[ph]
        nz = np.nonzero(cn)[0]
        if not len(nz):
            continue
        nch = nz.max() + 1
        c = cn[:nch]
        top = np.argsort(-c)[:12]
        print(f"phase {ph}: {nch} chunks, chunk ns median {np.median(c):.0f} p90 {np.percentile(c, 90):.0f} max {c.max()}")
        print("   slowest chunks (index, ns):", [(int(k), int(c[k])) for k in top])
        # mean by 100-chunk bucket
        b = [int(c[i:i + 500].mean()) for i in range(0, nch, 500)]
        print("   mean ns per 500-chunk bucket:", b)
