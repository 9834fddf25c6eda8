"""Generate the golden fixtures from the REFERENCE package (hornbp).

Run in the development container where /root/reference exists:

    python tests/golden/make_golden.py

It imports hornbp from /root/reference/pkg/src, rebuilds every BASELINE
configuration with the reference's own generator, compiler and engine, and
writes:

  tests/golden/golden.json         hashes + iteration counts + deltas (hex)
  tests/golden/weblech_c1.npz      full C1 marginals (small enough to commit)

The GPU box has no /root/reference, so the parity tests compare against
these files (and against the C oracle, which tests/test_oracle.py pins to
the same files).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sched_arrays(graph, schedule):
    """Reference Schedule -> canonical CSR arrays (edge index = rowptr[f] + slot)."""
    rp = np.zeros(graph.num_factors + 1, dtype=np.int64)
    np.cumsum([f.degree for f in graph.factors], out=rp[1:])
    out = []
    for batches in (schedule.s_batches, schedule.t_batches):
        off = np.zeros(len(batches) + 1, dtype=np.int64)
        np.cumsum([len(b) for b in batches], out=off[1:])
        idx = np.asarray([rp[e.factor] + e.slot for b in batches for e in b], dtype=np.int32)
        out += [off, idx]
    return out


def sched_sha(arrs) -> str:
    return hashlib.sha256(b"".join(np.ascontiguousarray(a).tobytes() for a in arrs)).hexdigest()


def residual_order_ref(hornbp, g):
    from hornbp.storage import initialize

    sched = hornbp.Strategy.parall().compile(g)
    store = initialize(g)
    before = store.ftov1 / (store.ftov0 + store.ftov1)
    hornbp.update_vtof_batch(store, list(sched.t_batches[0]))
    hornbp.update_ftov_batch(store, list(sched.s_batches[0]))
    after = store.ftov1 / (store.ftov0 + store.ftov1)
    r = np.abs(after - before)[store.vtof_to_ftov]
    return np.lexsort((np.arange(g.num_edges), -r))


def main() -> None:
    sys.path.insert(0, REF)
    import hornbp

    specs = {
        "weblech": (313, 383, 8, 0),
        "hedc": (1657, 3690, 8, 25),
        "avrora": (9424, 26667, 8, 3),
        "ftp": (101583, 109592, 8, 0),
    }
    gold: dict = {"generator": "hornbp (reference) via tests/golden/make_golden.py",
                  "numpy": np.__version__, "graphs": {}, "runs": {}, "sweep": {}}
    graphs = {}
    for name, spec in specs.items():
        g, alarms = hornbp.generate(hornbp.SynthSpec(*spec))
        graphs[name] = (g, alarms)
        gold["graphs"][name] = dict(
            V=g.num_variables, E=g.num_edges, F=g.num_factors,
            fastfg_sha=hashlib.sha256(g.to_fastfg().encode()).hexdigest(),
            alarms_sha=sha(np.asarray(alarms.alarms, dtype=np.int64)),
            labels_sha=sha(np.asarray(alarms.labels, dtype=np.int8)),
            n_alarms=len(alarms))
        print(name, gold["graphs"][name], flush=True)

    def record(key, g, strategy, max_it, tol, order_sha=None):
        t0 = time.time()
        sched = strategy.compile(g)
        arrs = sched_arrays(g, sched)
        res = hornbp.run(g, sched, hornbp.EngineOptions(max_iterations=max_it, tolerance=tol))
        gold["runs"][key] = dict(
            k=sched.num_batches, sched_sha=sched_sha(arrs),
            updates_per_iteration=int(len(arrs[1]) + len(arrs[3])),
            max_iterations=max_it, tolerance=tol,
            iterations=res.iterations, converged=res.converged,
            deltas=[float(d).hex() for d in res.deltas],
            marginals_sha=sha(res.marginals), order_sha=order_sha)
        print(key, {k: v for k, v in gold["runs"][key].items() if k != "deltas"},
              f"{time.time() - t0:.1f}s", flush=True)
        return res

    g, _ = graphs["weblech"]
    res = record("C1", g, hornbp.Strategy.parall(), 100, 0.0)
    np.savez_compressed(os.path.join(HERE, "weblech_c1.npz"), marginals=res.marginals,
                        deltas=np.asarray(res.deltas))
    record("C1-tol", g, hornbp.Strategy.parall(), 1000, 1e-9)
    g, _ = graphs["hedc"]
    edges = g.edge_list()
    perm = np.random.default_rng(1234).permutation(g.num_edges)
    record("C2", g, hornbp.Strategy.seqfix([edges[i] for i in perm]), 1000, 1e-9)
    record("C2-canonical", g, hornbp.Strategy.seqfix(), 1000, 1e-9)
    g, _ = graphs["avrora"]
    order = residual_order_ref(hornbp, g)
    edges = g.edge_list()
    record("C3", g, hornbp.Strategy.seqfix([edges[i] for i in order]), 1000, 1e-6,
           order_sha=sha(order.astype(np.int64)))
    record("C3-PARALL", g, hornbp.Strategy.parall(), 1000, 1e-6)
    g, alarms = graphs["ftp"]
    res = record("C4-PARALL", g, hornbp.Strategy.parall(), 1000, 1e-9)
    gold["runs"]["C4-PARALL"]["top10"] = hornbp.rank_alarms(res.marginals, alarms)[:10]
    gold["runs"]["C4-PARALL"]["top100_sha"] = sha(
        np.asarray(hornbp.rank_alarms(res.marginals, alarms)[:100], dtype=np.int64))
    record("C4-SEQFIX", g, hornbp.Strategy.seqfix(), 1000, 1e-9)

    # C5: evidence sets j (clamped to ground truth), PARALL tol 1e-9
    for j in range(4):
        t0 = time.time()
        rng = np.random.default_rng(j)
        pick = np.sort(rng.choice(len(alarms), 8, replace=False))
        cur = g
        for i in pick.tolist():
            cur = hornbp.clamp_evidence(cur, alarms.alarms[i], alarms.labels[i])
        sched = hornbp.Strategy.parall().compile(cur)
        res = hornbp.run(cur, sched, hornbp.EngineOptions(max_iterations=1000, tolerance=1e-9))
        labeled = [alarms.alarms[i] for i in pick.tolist()]
        ranked = hornbp.rank_alarms(res.marginals, alarms, labeled)
        gold["sweep"][str(j)] = dict(
            pick=pick.tolist(), iterations=res.iterations, converged=res.converged,
            last_delta=float(res.last_delta).hex(), marginals_sha=sha(res.marginals),
            p1_sha=sha(np.ascontiguousarray(res.marginals[:, 1])),
            top10=ranked[:10], top100_sha=sha(np.asarray(ranked[:100], dtype=np.int64)))
        print("C5 set", j, gold["sweep"][str(j)]["iterations"], f"{time.time() - t0:.1f}s",
              flush=True)

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(gold, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
