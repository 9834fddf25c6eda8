"""Benchmark: edge-message updates/sec and time-to-convergence (BASELINE.json).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                [--workload sweep|c4|c4-seqfix] [--sets 1024]

Default workload, every N: configs[4] of BASELINE.json -- the ftp-scale
interactive-ranking sweep. The graph is SynthSpec(101583, 109592, 8, 0)
(211,175 V / 476,915 E, pinned by sha256 in tests/test_synth.py); evidence
set j clamps 8 alarms drawn with default_rng(j) to their ground-truth labels
(SURVEY.md 8(d) C5); PARALL, tol 1e-9, every set run to its own convergence
from uniform messages. The 1,024 sets are partitioned across the N ranks
(contiguous slices, one GPU each, graph replicated, no per-iteration
collective) and the per-set outputs -- iterations, P1 of the 8,152 alarms and
the device top-100 alarm ranking -- are gathered to rank 0 with NCCL at the
end of every step. A step is the whole sweep (strong scaling: total work
fixed as N grows).

  value       edge-message updates/s = sum over sets of (sum|s_i| + |t_i|) x
              iterations (cli.py:337-344 per set) / device time of the step,
              CUDA events on the stream the sweep and the gather run on, max
              over ranks. Inputs (graph, evidence) resident in HBM. The
              working set (~17 GB at N=1) is far larger than L2.
  e2e         the same metric through the public API every step:
              run_many (N=1) / run_many_distributed (N>1) with the evidence
              lists on the host -- H2D of the evidence, the sweep, the gather,
              D2H of the gathered results to rank 0 -- wall clock, max over ranks.
  roofline    the persistent sweep kernel: algorithmic bytes per launch
               / its CUDA-event duration, against the
              measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline (rank 0, N=1) the C oracle, a bit-exact restatement of
              hornbp's clamp + compile + run, one set per host core in
              parallel, on a bounded sample of the same sets.
  single_graph (rank 0, N=1) configs[3]: the ftp graph alone, PARALL, time
              to convergence (the persistent single-graph executor).

--workload c4 / c4-seqfix: the single-graph line as the headline instead.
--impl reference: the reference's CPU path (the C oracle port -- the
reference is pure Python/numpy and cannot run on the GPU box), all host
cores, on a bounded sample of the same sets; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
from typing import Optional
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edge-message updates/sec and time-to-convergence on ftp-scale graph (477k edges)"
UNIT = "edge-message updates/s"
TOPK = 100


def load_peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---- algorithmic bytes -------------------------------------------------

def single_bytes_per_iteration(graph, updates: int) -> int:
    """16(|S|+|T|) message writes + 3*16*E message reads
    + 16*V marginal write/prev read + 8*E int32 indices + 4(V+1) + 4(F+1)
    rowptrs + 17*F factor params."""
    V, F, E = graph.num_variables, graph.num_factors, graph.num_edges
    return 16 * updates + 48 * E + 16 * V + 8 * E + 4 * (V + 1) + 4 * (F + 1) + 17 * F


def sweep_set_bytes(graph, iterations: np.ndarray, max_iterations: int) -> np.ndarray:
    """Algorithmic DRAM bytes the persistent sweep kernel moves for one set
    that stops after n iterations (csrc/sweep.cu): factor side n times
    (iteration 1 writes every ftov message and reads nothing; later ones read
    and write the T non-unary slots), variable side n times (reads every ftov
    message, the evidence byte and -- after the first -- the previous P0,
    writes P0 and, unless the run hit max_iterations, the T vtof messages),
    plus the row / twin / parameter indices shared by the 32 sets of a warp."""
    V, F, E = graph.num_variables, graph.num_factors, graph.num_edges
    deg = np.diff(np.asarray(graph.rowptr, dtype=np.int64))
    T = int(deg[deg > 1].sum())
    n = np.asarray(iterations, dtype=np.int64)
    fac = 16 * E + (n - 1) * 32 * T
    var = n * (16 * E + V + 8 * V) + (n - 1) * 8 * V + (n - (n == max_iterations)) * 16 * T
    idx = n * ((4 * (V + 1) + 4 * E) + (4 * (F + 1) + 4 * E + 16 * F)) / 32.0
    return fac + var + idx


# ---- reference arm -------------------------------------------------------------------------

def oracle_sets(graph, sets, cores: int, max_it: int, tol: float):
    """Run evidence sets on the C oracle, one single-threaded run per host
    core concurrently (ctypes releases the GIL). Returns (updates, seconds)."""
    from oracle import orc

    def one(ev):
        fg = orc.clamp(graph, ev[0], ev[1])
        arrs = orc.parall_arrays(fg)
        o = orc.run(fg, arrs, max_it, tol, threads=1)
        return (len(arrs[1]) + len(arrs[3])) * o["iterations"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as pool:
        upd = sum(pool.map(one, sets))
    return upd, time.perf_counter() - t0


REF_SITE = os.path.join(ROOT, "baseline", "_ref")  # the UNMODIFIED reference (pip --target)
FTP_SPEC = (101583, 109592, 8, 0)


def cpu_model() -> str:
    """The host CPU model (lscpu's "Model name"), for the baseline record."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.strip().startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def loaded_repo_libs() -> list:
    """Shared objects of this repo mapped into the process (/proc/self/maps)."""
    out = set()
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                path = line.split()[-1] if len(line.split()) >= 6 else ""
                if path.endswith(".so") and os.path.realpath(path).startswith(os.path.realpath(ROOT)):
                    out.add(os.path.relpath(os.path.realpath(path), os.path.realpath(ROOT)))
    except OSError:
        pass
    return sorted(out)


def import_reference():
    """hornbp from baseline/_ref (installed from /root/reference with pip
    --target; it travels to the GPU box with the snapshot)."""
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    import hornbp

    return hornbp


def ref_flat(R, graph):
    """A hornbp FactorGraph as the flat arrays the C port reads (canonical
    factor-major edge order, graph.py:146-150): nothing of this repo's package."""
    from oracle import orc

    deg = [1 + len(f.body) for f in graph.factors]
    rowptr = np.zeros(len(deg) + 1, dtype=np.int64)
    np.cumsum(deg, out=rowptr[1:])
    vars_ = np.fromiter((v for f in graph.factors for v in (f.head, *f.body)), dtype=np.int32,
                        count=int(rowptr[-1]))
    kind = np.fromiter((1 if f.kind is R.FactorKind.OR else 0 for f in graph.factors),
                       dtype=np.int8, count=len(deg))
    p1 = np.fromiter((f.p1 for f in graph.factors), dtype=np.float64, count=len(deg))
    p2 = np.fromiter((f.p2 for f in graph.factors), dtype=np.float64, count=len(deg))
    return orc.FlatGraph(graph.num_variables, rowptr, vars_, kind, p1, p2)


def ref_evidence_set(alarms, j: int, size: int = 8):
    """C5 set j: default_rng(j).choice(#alarms, 8), sorted,
    clamped to the ground-truth labels."""
    pick = np.sort(np.random.default_rng(j).choice(len(alarms), size, replace=False))
    return (np.asarray(alarms.alarms, dtype=np.int64)[pick],
            np.asarray(alarms.labels, dtype=bool)[pick])


def ref_schedule_arrays(R, graph, sched):
    """A hornbp Schedule as (s_off, s_edges, t_off, t_edges) canonical indices."""
    rp = np.zeros(len(graph.factors) + 1, dtype=np.int64)
    np.cumsum([1 + len(f.body) for f in graph.factors], out=rp[1:])

    def flat(batches):
        off = np.zeros(len(batches) + 1, dtype=np.int64)
        np.cumsum([len(b) for b in batches], out=off[1:])
        idx = np.fromiter((rp[e.factor] + e.slot for b in batches for e in b), dtype=np.int32,
                          count=int(off[-1]))
        return off, idx

    s_off, s_e = flat(sched.s_batches)
    t_off, t_e = flat(sched.t_batches)
    return s_off, s_e, t_off, t_e


def python_reference(R, graph, alarms, cores: int) -> dict:
    """The reference's own Python engine: hornbp.run on the ftp
    graph under PARALL, best of 3 with workers=1 (its fastest setting) and once
    with workers=cores; plus one C5 set end to end through the reference API
    (8 x clamp_evidence + compile + run + rank_alarms)."""
    opts = R.EngineOptions(max_iterations=1000, tolerance=1e-9)
    t0 = time.perf_counter()
    sched = R.Strategy.parall().compile(graph)
    compile_s = time.perf_counter() - t0
    upd = sum(len(b) for b in sched.s_batches) + sum(len(b) for b in sched.t_batches)
    best, its = None, 0
    for _ in range(3):
        t0 = time.perf_counter()
        r = R.run(graph, sched, opts, workers=1)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        its = r.iterations
    t0 = time.perf_counter()
    r = R.run(graph, sched, opts, workers=cores)
    many = time.perf_counter() - t0
    ids, labels = ref_evidence_set(alarms, 0)
    t0 = time.perf_counter()
    cur = graph
    for v, lab in zip(ids.tolist(), labels.tolist()):
        cur = R.clamp_evidence(cur, int(v), bool(lab))
    s0 = R.Strategy.parall().compile(cur)
    r0 = R.run(cur, s0, opts, workers=1)
    R.rank_alarms(r0.marginals, alarms, ids.tolist())
    set_s = time.perf_counter() - t0
    upd0 = sum(len(b) for b in s0.s_batches) + sum(len(b) for b in s0.t_batches)
    return {
        "impl": "hornbp (the reference package, baseline/_ref), pure Python/numpy",
        "c4_parall": {"iterations": its, "updates_per_iteration": upd, "compile_s": compile_s,
                      "run_s_workers1_best_of_3": best, "updates_per_s_workers1": upd * its / best,
                      "run_s_workers_cores": many, "workers_cores": cores,
                      "updates_per_s_workers_cores": upd * its / many},
        "c5_set0_end_to_end": {"seconds": set_s, "iterations": r0.iterations,
                               "updates_per_s": upd0 * r0.iterations / set_s,
                               "what": "8 x clamp_evidence + Strategy.parall().compile + run "
                                       "(workers=1) + rank_alarms, one set, serial"},
    }


def run_reference(args) -> None:
    """The reference arm. Imports nothing from this repo's package: the graph
    and evidence come from the reference's own generator (hornbp.synth, from
    baseline/_ref), the timed engine is the C port of hornbp's CPU path
    (oracle/, pinned bit-for-bit to hornbp), and the reference's own Python
    engine is timed beside it."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import orc

    R = import_reference()
    cores = os.cpu_count() or 1
    graph, alarms = R.generate(R.SynthSpec(*FTP_SPEC))
    fg = ref_flat(R, graph)
    if args.workload in ("c4", "c4-seqfix"):
        key = "C4-SEQFIX" if args.workload == "c4-seqfix" else "C4-PARALL"
        strat = R.Strategy.seqfix() if args.workload == "c4-seqfix" else R.Strategy.parall()
        arrs = ref_schedule_arrays(R, graph, strat.compile(graph))
        upd = len(arrs[1]) + len(arrs[3])
        for _ in range(args.warmup):
            orc.run(fg, arrs, 1000, 1e-9, threads=cores)
        times, iters = [], []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            o = orc.run(fg, arrs, 1000, 1e-9, threads=cores)
            times.append(time.perf_counter() - t0)
            iters.append(o["iterations"])
        value = upd * sum(iters) / sum(times)
        config = {"workload": f"{key}: ftp SynthSpec(101583,109592,8,0), "
                              f"{'SEQFIX' if 'SEQ' in key else 'PARALL'}, tol 1e-9, run to convergence",
                  "iterations": iters[-1], "updates_per_iteration": upd}
        sample = f"{args.steps} full {key} runs (C port, OpenMP over {cores} threads)"
        ms = 1e3 * sum(times) / args.steps
    else:
        n = args.sets
        per_step = cores  # one set per core per step: a bounded sample of the sweep
        steps_sets = [[ref_evidence_set(alarms, (k * per_step + i) % n) for i in range(per_step)]
                      for k in range(args.warmup + args.steps)]
        for k in range(args.warmup):
            oracle_sets(fg, steps_sets[k], cores, 1000, 1e-9)
        tot_upd, tot_s = 0, 0.0
        for k in range(args.warmup, args.warmup + args.steps):
            u, s_ = oracle_sets(fg, steps_sets[k], cores, 1000, 1e-9)
            tot_upd += u
            tot_s += s_
        value = tot_upd / tot_s
        config = sweep_config(n, args.gpus)
        sample = (f"{args.steps} steps x {per_step} evidence sets (sets "
                  f"{args.warmup * per_step % n}..), one set per core, C port single-threaded runs "
                  "(clamp + PARALL compile + run)")
        ms = 1e3 * tot_s / args.steps
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if args.workload == "sweep" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (hornbp.synth.generate, the "
        "reference's own generator)", "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if os.environ.get("HBP_BENCH_NO_PYREF") != "1":
        line["python_reference"] = python_reference(R, graph, alarms, cores)
    # the arm must not have touched the product (its native library included)
    assert not any(m.split(".")[0] == "paper_2509_22337_b200" for m in sys.modules), \
        "reference arm imported the product package"
    line["native_libs_loaded"] = loaded_repo_libs()
    print(json.dumps(line), flush=True)


def sweep_config(n_sets: int, n_gpus: int) -> dict:
    return {"workload": f"C5 ftp interactive-ranking sweep: {n_sets} evidence sets x 8 clamped "
                        "alarms over SynthSpec(101583,109592,8,0) (211,175 V / 476,915 E), "
                        "PARALL, tol 1e-9, each set to its own convergence from uniform",
            "sets": n_sets, "evidence_per_set": 8, "outputs": f"iterations + P1 of 8,152 alarms "
            f"+ device top-{TOPK} ranking per set, NCCL-gathered to rank 0",
            "parallelism": f"sets sharded over {n_gpus} GPU(s), graph replicated",
            "l2": "working set > L2 (17 GB of messages at N=1); no flush needed"}


# ---- our arm: the sweep ------------------------------------------------------------------------

def run_ours_sweep(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2509_22337_b200 as P
    from paper_2509_22337_b200 import distributed as D
    from paper_2509_22337_b200 import workloads as W

    world, rank, local = dist_env()
    # HBP_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0 with gloo --
    # exercises the multi-rank path on a one-GPU box; NCCL refuses shared GPUs
    shared = os.environ.get("HBP_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    P.engine.set_device(local)
    multi = world > 1
    if multi:
        # NCCL's init lines (nranks, NVLS) go to stderr: the driver's log shows
        # the communicator; stdout stays the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    g, alarms = W.graph("ftp")
    n = args.sets
    sets = [W.evidence_set(alarms, j) for j in range(n)]
    sel = np.sort(np.asarray(alarms.alarms, dtype=np.int32))
    lo, hi = D.partition(n, world, rank)
    # the rank's evidence sets as host CSR arrays, built once (like any input
    # resident in host memory); every step still uploads them
    mine = P.EvidenceCSR.from_sets(g, sets[lo:hi])
    m = hi - lo
    opts = P.EngineOptions(1000, 1e-9)
    p1 = torch.empty((m, len(sel)), dtype=torch.float64, device=dev)
    rk = torch.empty((m, TOPK), dtype=torch.int32, device=dev)
    dg = P.engine.device_graph(g)
    stream = torch.cuda.current_stream(dev)
    dg.set_stream(stream)

    def step():
        r = P.run_many(g, mine, None, opts, marginals=False, deltas=False, select=sel, topk=TOPK,
                       device_out={"p1_select": p1, "ranked": rk})
        if multi:
            D.gather_rows(torch, dist, p1, n, world, rank)
            D.gather_rows(torch, dist, rk, n, world, rank)
            st = torch.as_tensor(r.iterations, device=dev).reshape(-1, 1)
            D.gather_rows(torch, dist, st, n, world, rank)
        return r

    for _ in range(args.warmup):
        step()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            results.append(step())
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    upd_local = sum(r.total_updates() for r in results)
    kernel_ms = [r.kernel_ms for r in results]
    launches = sum(r.launches for r in results) + (3 * args.steps if multi else 0)
    t = torch.tensor([ms, float(upd_local)], dtype=torch.float64, device=dev)
    if multi:
        mx = t[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t[1:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, upd_total = float(mx.item()), float(sm.item())
    else:
        ms_max, upd_total = ms, float(upd_local)
    value = upd_total / (ms_max * 1e-3)
    dg.set_stream(None)

    # parity of the benchmarked outputs against the reference's golden C5 sets
    parity = None
    if rank == 0:
        try:
            import hashlib
            with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
                gold = json.load(fh)["sweep"]
            ok = True
            for j in range(min(4, m)):
                want = gold[str(j)]
                ok &= int(results[-1].iterations[j]) == want["iterations"]
                ok &= rk[j, :10].cpu().tolist() == want["top10"]
                ok &= hashlib.sha256(rk[j].cpu().numpy().astype(np.int64).tobytes()
                                     ).hexdigest() == want["top100_sha"]
            parity = bool(ok)
        except (OSError, KeyError):
            pass

    # ---- end to end through the public API (host evidence in, host results out) ----
    e2e_s = []
    h2d = d2h = 0
    for i in range(args.warmup + args.steps):
        if multi:
            dist.barrier()
        t0 = time.perf_counter()
        if multi:
            out = D.run_many_distributed(g, sets, opts, select=sel, topk=TOPK)
            upd_e2e = float(out.total_updates()) if rank == 0 else 0.0
        else:
            out = P.run_many(g, sets, None, opts, marginals=False, deltas=False, select=sel,
                             topk=TOPK)
            upd_e2e = float(out.total_updates())
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_s.append(dt)
    tt = torch.tensor([sum(e2e_s)], dtype=torch.float64, device=dev)
    if multi:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_value = upd_e2e * len(e2e_s) / float(tt.item())
    nev = 8 * m
    h2d = 8 * (m + 1) + 5 * nev + 4 * len(sel)
    # per-set control words read back by every rank + (rank 0) the gathered results
    max_it_seen = int(max(int(r.iterations.max()) for r in results)) if m else 0
    ctrl = 8 * m + 20 * (max_it_seen + 2) * ((m + 31) // 32 * 32)
    d2h = ctrl + (n * (8 * len(sel) + 4 * TOPK + 40) if rank == 0 else 0)

    if rank != 0:
        if multi:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the persistent sweep kernel (rank 0) ----
    peak, peak_kind = load_peaks()
    last = results[-1]
    bytes_launch = float(sweep_set_bytes(g, last.iterations, 1000).sum())
    achieved = bytes_launch / (statistics.mean(kernel_ms) * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tj = json.load(fh)
        if tj.get("kernel") == "sweep_ws" and tj.get("sets") == m:
            traffic = float(tj["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        pass

    cfg = sweep_config(n, world)
    if shared and multi:
        cfg["shared_gpu"] = (f"test mode: all {world} ranks on cuda:0 over gloo "
                             "(HBP_BENCH_SHARED_GPU=1, the box has fewer GPUs than ranks)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "time_to_convergence_ms": ms_max / args.steps,
        "iterations": {"min": int(last.iterations.min()), "max": int(last.iterations.max()),
                       "mean": float(last.iterations.mean())},
        "parity_vs_reference_golden": parity,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * float(tt.item()) / len(e2e_s),
                "path": ("paper_2509_22337_b200.run_many_distributed" if multi else
                         "paper_2509_22337_b200.run_many") + " with host evidence (CSR arrays)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}), burst copy",
                     "kernel": "hbp::sweep_ws<1,1> (rank 0's whole slice in one launch)",
                     "bytes_per_launch": bytes_launch, "sets_per_launch": m,
                     "kernel_ms": statistics.mean(kernel_ms)},
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    if not multi:
        cores = os.cpu_count() or 1
        sample = [sets[j] for j in range(min(n, cores))]
        u, s = oracle_sets(g, sample, cores, 1000, 1e-9)
        line["cpu_baseline"] = {"value": u / s, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"sets 0..{len(sample) - 1}, one per core, C oracle "
                                          "single-threaded runs (clamp + PARALL compile + run)"}
        line["fp32_mode"] = measure_fp32(P, g, sets, sel, p1.cpu().numpy(), rk.cpu().numpy())
        line["single_graph"] = measure_single(torch, "C4-PARALL", steps=20, warmup=5)
        # every other BASELINE configuration on the same line (configs[0..3])
        line["configs"] = {k: measure_single(torch, k, steps=10, warmup=3)
                           for k in SINGLE_KEYS if k != "C4-PARALL"}
        line["interaction_loop"] = measure_loop(g, alarms, cores)
    print(json.dumps(line), flush=True)
    if multi:
        dist.barrier()
        dist.destroy_process_group()


# ---- optional fp32 mode ------------------------------------------------

def measure_fp32(P, g, sets, sel, p1_64, rk_64) -> dict:
    """The same sweep with fp32 message storage (fp64 arithmetic and
    marginals), against this run's fp64 outputs: north-star bar 1e-5."""
    opts = P.EngineOptions(1000, 1e-9, precision="fp32")
    P.run_many(g, sets[:64], None, opts, marginals=False, deltas=False)
    ks, last = [], None
    for _ in range(3):
        last = P.run_many(g, sets, None, opts, marginals=False, deltas=False, select=sel, topk=TOPK)
        ks.append(last.kernel_ms)
    k = min(ks)
    return {"value": last.total_updates() / (k * 1e-3), "unit": UNIT, "kernel_ms": k,
            "dtype": "f32 messages, f64 arithmetic and marginals",
            "max_abs_p1_diff_vs_f64": float(np.abs(last.p1_select - p1_64).max()),
            "top100_identical_sets": int((last.ranked == rk_64).all(axis=1).sum()),
            "sets": len(sets)}


# ---- device-resident interaction loop ------------------------------------

def measure_loop(g, alarms, cores: int) -> dict:
    """ranking.interaction_loop on the ftp graph under PARALL until every true
    alarm is revealed (the paper's TotalTime), next to the
    reference's per-round cost (clamp + compile + run) sampled on the oracle."""
    import paper_2509_22337_b200 as P
    from oracle import orc

    opts = P.EngineOptions(1000, 1e-9)
    P.interaction_loop(g, alarms, P.Strategy.parall(), opts, max_rounds=3)
    t0 = time.perf_counter()
    tr = P.interaction_loop(g, alarms, P.Strategy.parall(), opts)
    total = time.perf_counter() - t0
    m = P.compute_metrics(tr)
    # reference round sample: rounds 1..3 of the same trace on the oracle
    labeled_v, labeled_l, ref_s = [], [], []
    for rnd in tr.rounds[:3]:
        t1 = time.perf_counter()
        fg = orc.clamp(g, labeled_v, labeled_l)
        o = orc.run(fg, orc.parall_arrays(fg), 1000, 1e-9, threads=cores)
        ref_s.append(time.perf_counter() - t1)
        assert o["marginals"][rnd.alarm, 1] == rnd.p_true
        labeled_v.append(rnd.alarm)
        labeled_l.append(rnd.label)
    ref_round = statistics.mean(ref_s)
    return {"workload": "ftp PARALL, tol 1e-9: rank -> reveal the top alarm -> clamp -> rerun "
                        "from uniform, until every true alarm is revealed (ranking.py:94-135)",
            "rounds": len(tr.rounds), "total_s": total, "ms_per_round": 1e3 * total / len(tr.rounds),
            "metrics": {"rank_100t": m.rank_100t, "rank_90t": m.rank_90t,
                        "inversions": m.inversions, "auc": m.auc},
            "reference_ms_per_round": 1e3 * ref_round,
            "reference_total_s_estimate": ref_round * len(tr.rounds),
            "reference_kind": f"C oracle port (clamp + PARALL compile + run), {cores} threads, "
                              "rounds 1-3 sampled, p_true bit-checked",
            "path": "paper_2509_22337_b200.interaction_loop (evidence codes + device ranking)"}


# ---- single graphs (configs[0..3]) ---------------------------------------------------------

SINGLE_KEYS = ("C1", "C2", "C3", "C4-PARALL", "C4-SEQFIX")
WORKLOAD_TEXT = {
    "C1": "C1: weblech SynthSpec(313,383,8,0) (696 V / 1,655 E), PARALL, fixed 100 iterations",
    "C2": "C2: hedc SynthSpec(1657,3690,8,25) (5,347 V / 14,231 E), user-defined sequential sweep "
          "(SEQFIX over default_rng(1234).permutation(E), 224 levels), tol 1e-9",
    "C3": "C3: avrora SynthSpec(9424,26667,8,3) (36,091 V / 100,789 E), static residual-priority "
          "order (SEQFIX, 303 levels), tol 1e-6",
    "C4-PARALL": "C4-PARALL: ftp SynthSpec(101583,109592,8,0) (211,175 V / 476,915 E), PARALL, tol 1e-9",
    "C4-SEQFIX": "C4-SEQFIX: ftp SynthSpec(101583,109592,8,0), canonical SEQFIX (476 levels), tol 1e-9",
}


def plan_info(lib, plan) -> tuple[int, int, int, int]:
    import ctypes as C
    f = lib.hbp_debug_plan_info
    f.restype = None
    f.argtypes = [C.c_void_p] + [C.POINTER(C.c_int32)] * 4
    v = [C.c_int32() for _ in range(4)]
    f(plan.handle, *[C.byref(x) for x in v])
    return tuple(x.value for x in v)  # phases, grid, threads, fused levels


def l2_traffic(key: str) -> Optional[dict]:
    """lts__t_sectors of one launch of this config's kernel, from this round's
    ncu capture (profiles/l2_traffic.json, written by tools/collect_l2.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "l2_traffic.json")) as fh:
            return json.load(fh).get(key)
    except (OSError, ValueError):
        return None


def measure_single(torch, key: str, steps: int, warmup: int, e2e: bool = True,
                   cpu: bool = True) -> dict:
    """One single-graph config: device time to convergence (CUDA events
    around the one persistent launch, L2 flushed before each run), updates/s,
    roofline, parity against the reference's golden run, the public run()
    end to end, and the C port on one host core."""
    import ctypes as C

    import paper_2509_22337_b200 as P
    from oracle import orc
    from paper_2509_22337_b200 import _native
    from paper_2509_22337_b200 import workloads as W

    w = W.build(key)
    g = w.graph
    sched = w.strategy.compile(g)
    opts = P.EngineOptions(max_iterations=w.max_iterations, tolerance=w.tolerance)
    upd = sched.updates_per_iteration()
    flush = torch.empty(256 << 20 >> 2, dtype=torch.float32, device="cuda")
    lib = _native.lib()
    dg = P.engine.device_graph(g)
    plan = dg.plan(sched, g)
    copt = plan.options(opts)
    nphases, grid, threads, nfused = plan_info(lib, plan)
    lib.hbp_debug_plan_pslot.restype = C.c_int32
    lib.hbp_debug_plan_pslot.argtypes = [C.c_void_p]
    pslot = lib.hbp_debug_plan_pslot(plan.handle) == 1
    kernel = ("hbp::lbp_pslot (PARALL, one phase per iteration; whole run in one launch)" if pslot
              else "hbp::lbp_persistent (whole run in one launch)")

    def step():
        res = _native.Result()
        st = lib.hbp_run_device(plan.handle, C.byref(copt), C.byref(res), None)
        if st != 0:
            raise RuntimeError(_native.last_error())
        return res

    for _ in range(max(3, warmup)):
        step()
    dev_ms, iters, launches = [], [], 0
    torch.cuda.synchronize()
    for _ in range(steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        r = step()
        dev_ms.append(r.device_ms)
        iters.append(r.iterations)
        launches += lib.hbp_last_launch_count()
    total_ms = sum(dev_ms)
    value = upd * sum(iters) / (total_ms * 1e-3)
    res_check = P.run(g, sched, opts)
    parity = None
    try:
        import hashlib
        with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
            gold = json.load(fh)["runs"][key]
        parity = (hashlib.sha256(res_check.marginals.tobytes()).hexdigest() == gold["marginals_sha"]
                  and res_check.iterations == gold["iterations"]
                  and [float(d).hex() for d in res_check.deltas] == gold["deltas"])
    except (OSError, KeyError):
        pass
    E, V, F = g.num_edges, g.num_variables, g.num_factors
    peak, peak_kind = load_peaks()
    bpi = single_bytes_per_iteration(g, upd)
    mean_ms = statistics.mean(dev_ms)
    bytes_per_launch = bpi * statistics.mean(iters) + 32 * E
    achieved = bytes_per_launch / (mean_ms * 1e-3) / 1e9
    l2 = l2_roofline(achieved)
    levelled = sched.num_batches > 1
    out = {
        "workload": WORKLOAD_TEXT[key] + ", to convergence, L2 flushed (256 MiB write) between runs",
        "value": value, "unit": UNIT, "time_to_convergence_ms": total_ms / steps,
        "iterations": iters[-1], "updates_per_iteration": upd, "k_batches": sched.num_batches,
        "phases_per_iteration": 1 if pslot else nphases, "fused_levels": nfused,
        "grid": [grid, threads],
        "parity_vs_reference_golden": parity, "gpu_launches": launches,
    }
    if levelled or key == "C1":
        # dependent-chain latency, not bandwidth: each phase is a barrier-
        # separated dependent step (a level on CTA 0, or a whole-graph pass)
        out["roofline"] = {
            "bound": "latency",
            "us_per_phase": 1e3 * mean_ms / (iters[-1] * (1 if pslot else nphases)),
            "phases": iters[-1] * (1 if pslot else nphases), "achieved_gbs": achieved,
            "hbm_frac": achieved / peak, "l2_frac": l2["frac"] if l2 else None,
            "kernel": kernel,
            "bytes_per_launch": bytes_per_launch}
    else:
        tr = l2_traffic(key)
        out["roofline"] = {
            "bound": "l2", "achieved": achieved, "peak": l2["peak"] if l2 else None,
            "unit": "GB/s", "frac": l2["frac"] if l2 else None,
            "traffic": tr["l2_bytes_per_launch"] if tr else None,
            "traffic_source": tr["source"] if tr else None,
            "peak_source": l2["peak_source"] if l2 else None,
            "hbm": {"peak": peak, "frac": achieved / peak,
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
            "kernel": kernel,
            "bytes_per_launch": bytes_per_launch,
            "note": "working set (~36 MB) is L2-resident within a run; algorithmic bytes are "
                    "SURVEY.md 8(d)'s two-phase count (lbp_pslot moves about the same: it "
                    "re-reads variable rows instead of writing and reading vtof messages)"}
    if e2e:
        # end to end through run(): fresh device layout + plan every step. The
        # graphs and sweeps of the earlier legs are released (and collected)
        # first, so their multi-GB frees do not land inside a timed step.
        import gc
        P.engine.clear_device_cache()
        gc.collect()
        torch.cuda.synchronize()
        e2e_s, e2e_iters = [], []
        for i in range(max(5, warmup) + steps):
            P.engine.clear_device_cache()
            t0 = time.perf_counter()
            r = P.run(g, sched, opts)
            dt = time.perf_counter() - t0
            if i >= max(5, warmup):
                e2e_s.append(dt)
                e2e_iters.append(r.iterations)
        s_off, s_e, t_off, t_e = sched.arrays(g)
        # canonical graph (rowptr, vars, kind, p1, p2) -> device layout build, then
        # the schedule's batches -> device PARALL shape test / host level plan
        h2d = 8 * (F + 1) + 4 * E + 17 * F + 4 * (len(s_e) + len(t_e))
        d2h = 16 * V + 8 * e2e_iters[-1]
        out["e2e"] = {"value": upd * sum(e2e_iters) / sum(e2e_s), "unit": UNIT,
                      "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                      "ms_per_step": 1e3 * statistics.mean(e2e_s),
                      "path": "paper_2509_22337_b200.run() with a fresh graph every step "
                              "(device layout build + plan + run + marginals to host)"}
    if cpu:
        t0 = time.perf_counter()
        o = orc.run(g, sched.arrays(g), w.max_iterations, w.tolerance, threads=1)
        cpu_s = time.perf_counter() - t0
        assert o["marginals"].tobytes() == res_check.marginals.tobytes()
        out["cpu_baseline"] = {"value": upd * o["iterations"] / cpu_s, "unit": UNIT, "cores": 1,
                               "kind": "port", "seconds": cpu_s,
                               "sample": f"one full {key} run, C oracle single-threaded "
                                         "(bit-identical marginals checked)"}
    return out


def l2_roofline(achieved: float) -> Optional[dict]:
    """The same algorithmic rate against the measured L2 read+write bandwidth
    (profiles/l2_peak.json, tools/l2_bench.cu; SURVEY.md 8(d) asks for it)."""
    try:
        with open(os.path.join(ROOT, "profiles", "l2_peak.json")) as fh:
            runs = json.load(fh)["runs"]
    except (OSError, KeyError, ValueError):
        return None
    peak = max(r["read_write_gbs"] for r in runs)
    return {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": "profiles/l2_peak.json: best L2-resident 16-B read+write stream (tools/l2_bench.cu)"}


def run_ours_single(args) -> None:
    import torch

    torch.cuda.set_device(0)
    import paper_2509_22337_b200 as P

    P.engine.set_device(0)
    key = {"c4": "C4-PARALL", "c4-seqfix": "C4-SEQFIX", "c1": "C1", "c2": "C2",
           "c3": "C3"}[args.workload]
    with ClockSampler(0) as clk:
        sg = measure_single(torch, key, args.steps, args.warmup)
    line = {
        "metric": METRIC, "value": sg["value"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sg["time_to_convergence_ms"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": sg["workload"], "iterations": sg["iterations"],
                   "updates_per_iteration": sg["updates_per_iteration"],
                   "k_batches": sg["k_batches"], "parallelism": "single graph, 1 GPU"},
        "time_to_convergence_ms": sg["time_to_convergence_ms"],
        "parity_vs_reference_golden": sg["parity_vs_reference_golden"],
        "e2e": sg["e2e"], "roofline": sg["roofline"], "cpu_baseline": sg["cpu_baseline"],
        "clocks": clk.summary(), "gpu_launches": sg["gpu_launches"],
    }
    print(json.dumps(line), flush=True)


def spawn(args) -> None:
    """`python bench.py --gpus N` outside torchrun: launch the N ranks the
    way the driver does (torch.distributed.run, one process per GPU, rendezvous
    on 127.0.0.1). On a box with fewer than N GPUs the ranks share cuda:0 over
    gloo (HBP_BENCH_SHARED_GPU=1, a test mode the JSON line names)."""
    import socket

    import torch

    env = dict(os.environ)
    if torch.cuda.device_count() < args.gpus:
        env["HBP_BENCH_SHARED_GPU"] = "1"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd, env=env).returncode)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["sweep", "c1", "c2", "c3", "c4", "c4-seqfix"],
                    default="sweep")
    ap.add_argument("--sets", type=int, default=1024)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload == "sweep":
        run_ours_sweep(args)
    else:
        run_ours_single(args)


if __name__ == "__main__":
    main()
