"""Scratch probe (GPU box): per-phase timeline from HBP_TRACE=1 (phase compute vs barrier)."""
import ctypes as C, os, sys, time
os.environ["HBP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_22337_b200 as P
from paper_2509_22337_b200 import _native, workloads as W
name = sys.argv[1]
wl = W.build(name)
w = wl
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
lib.hbp_debug_plan_info(plan.handle, C.byref(nph), C.byref(grid), C.byref(thr), None)
nph, G = nph.value, grid.value
n = 4 * nph * G * 2 + 2 * 16384
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
if d1 is not None:
    m1 = d1.mean(0)
    o1 = np.argsort(-m1)
    print("phase-1 slowest CTAs (cta, sm, mean us):", [(int(c), int(smid[c]), round(float(m1[c]), 2)) for c in o1[:8]])
    print("phase-1 median %.2f us" % np.median(m1))
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

# per-warp totals under the boustrophedon map, and what an LPT round->warp
# map (measured round costs) would give
if chunk_ns is not None:
    import heapq
    wpc = thr.value // 32
    for ph in range(2):
        cn = chunk_ns[ph]
        nz = np.nonzero(cn)[0]
        if not len(nz):
            continue
        nch = nz.max() + 1
        c = cn[:nch].astype(np.float64)
        R = -(-nch // G)
        tot = np.zeros((G, wpc))
        for k in range(nch):
            r, p = divmod(k, G)
            b = p if r % 2 == 0 else G - 1 - p
            tot[b, r % wpc] += c[k]
        rc = np.array([c[r * G:(r + 1) * G].mean() for r in range(R)])
        rmax = np.array([c[r * G:(r + 1) * G].max() for r in range(R)])
        # LPT: rounds by cost desc onto the least-loaded warp
        heap = [(0.0, w) for w in range(wpc)]
        assign = {}
        for r in np.argsort(-rc):
            load, w = heapq.heappop(heap)
            assign[r] = w
            heapq.heappush(heap, (load + rc[r], w))
        tot2 = np.zeros((G, wpc))
        for k in range(nch):
            r, p = divmod(k, G)
            b = p if r % 2 == 0 else G - 1 - p
            tot2[b, assign[r]] += c[k]
        print(f"phase {ph}: rounds {R}, warp totals now: max {tot.max()/1e3:.2f} us, per-CTA max-warp median {np.median(tot.max(1))/1e3:.2f}; "
              f"LPT rounds: max {tot2.max()/1e3:.2f} us, per-CTA median {np.median(tot2.max(1))/1e3:.2f}; ideal mean {tot.sum()/G/wpc/1e3:.2f}")

# chunk cost by item class (pure chunks only): the cost model's input
if chunk_ns is not None:
    g = wl.graph
    vdeg = np.bincount(np.asarray(g.vars), minlength=g.num_variables)
    fdeg = np.diff(np.asarray(g.rowptr))
    fkind = np.asarray(g.kind)
    K = 4
    # phase 0 items
    hv = np.sort(vdeg[vdeg > K])
    items0 = np.concatenate([np.repeat(hv, hv) + 1000, np.sort(vdeg[vdeg <= K])])  # +1000 marks heavy slots
    # phase 1 items: heavy AND slots, heavy OR slots, light AND nodes, light OR nodes
    hA = np.sort(fdeg[(fdeg > K) & (fkind == 0)]); hO = np.sort(fdeg[(fdeg > K) & (fkind == 1)])
    lA = np.sort(fdeg[(fdeg <= K) & (fkind == 0)]); lO = np.sort(fdeg[(fdeg <= K) & (fkind == 1)])
    items1 = np.concatenate([np.repeat(hA, hA) + 1000, np.repeat(hO, hO) + 2000, lA, lO + 100])
    for ph, items in ((0, items0), (1, items1)):
        c = chunk_ns[ph][: -(-len(items) // 32)].astype(np.float64)
        cls = {}
        for k in range(len(c)):
            u = np.unique(items[32 * k: 32 * k + 32])
            key = tuple(int(x) for x in u)
            cls.setdefault(key, []).append(c[k])
        rows = sorted(cls.items(), key=lambda kv: kv[0])
        print(f"phase {ph} class costs (item code: deg, +100 OR light, +1000 heavy AND/var slot, +2000 heavy OR slot):")
        print("   " + "; ".join(f"{k}: n={len(v)} {np.mean(v):.0f}" for k, v in rows if len(v) >= 1))

# levelled schedules: CTA 0's per-phase compute time distribution (small levels)
if nph > 8:
    d0 = (a[1, :, 0, 1] - a[1, :, 0, 0]) / 1e3
    d0 = d0[a[1, :, 0, 0] > 0]
    typ = np.arange(len(d0)) % 2
    for t in (0, 1):
        x = d0[2:][typ[2:] == t]
        print(f"CTA0 small phases type {t}: n={len(x)} min {x.min():.2f} p10 {np.percentile(x,10):.2f} "
              f"median {np.median(x):.2f} p90 {np.percentile(x,90):.2f} max {x.max():.2f} us")
