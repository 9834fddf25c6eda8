"""Copy one gpu_round2.sh output (gpurun_out/<tag>) into profiles/ as round-2 evidence:
bench lines (ours + reference arm), the bench launch list (CSV + per-kernel summary),
the sweep kernel's full capture (DRAM traffic -> profiles/traffic.json, read by bench.py)
and the single-graph kernels' full captures (L2 sectors -> profiles/l2_traffic.json,
read by bench.py). Usage: python tools/collect_r2.py <tag> [prefix=r2]"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
pre = sys.argv[2] if len(sys.argv) > 2 else "r2"
src = os.path.join(ROOT, "gpurun_out", tag)
prof = os.path.join(ROOT, "profiles")

SCALE = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2]


def metric(hdr, units, vals, name, want="byte"):
    i = hdr.index(name)
    v = float(vals[i].replace(",", ""))
    u = units[i]
    if want == "byte":
        return v * SCALE.get(u, 1.0)
    if want == "ms":
        return v * SCALE.get(u, 1.0)
    return v


def stall_mix(hdr, vals):
    st = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(vals[i] or 0)
          for i, n in enumerate(hdr)
          if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
    return ", ".join(f"{k} {100 * x / tot:.1f} %" for k, x in top)


def summary(rep):
    h, u, v = raw(rep)
    get = lambda n, w="x": metric(h, u, v, n, w)
    return {
        "duration_ms": get("gpu__time_duration.sum", "ms"),
        "dram_bytes": get("dram__bytes_read.sum", "byte") + get("dram__bytes_write.sum", "byte"),
        "l2_sectors": get("lts__t_sectors.sum"),
        "l1_ld_sectors": get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
        "l1_st_sectors": get("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum"),
        "inst": get("smsp__inst_executed.sum"),
        "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "regs": get("launch__registers_per_thread"),
        "dram_pct": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") if "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed" in h else get("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        "lts_pct": get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "stalls": stall_mix(h, v),
        "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "",
    }


bench = json.load(open(os.path.join(src, "bench.json")))
json.dump(bench, open(os.path.join(prof, f"{pre}_bench_n1.json"), "w"), indent=1)
ref = json.load(open(os.path.join(src, "bench_ref.json")))
json.dump(ref, open(os.path.join(prof, f"{pre}_bench_ref_n1.json"), "w"), indent=1)

# ---- launch list
rawl = open(os.path.join(src, "launches.csv")).read()
open(os.path.join(prof, f"{pre}_bench_launches.csv"), "w").write(rawl)
rows = [r for r in csv.reader(io.StringIO(rawl)) if len(r) > 5][1:]
agg = collections.OrderedDict()
for r in rows:
    a = agg.setdefault(r[4], [0, 0.0])
    a[0] += 1
    a[1] += float(r[-1].replace(",", "")) / 1e6
tot = sum(a[1] for a in agg.values()) or 1.0
lines = [f"# {pre} -- launch list of `python bench.py --steps 2 --warmup 3`", "",
         "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 3`",
         f"(cold-cache, serialised per-launch times: compare shares, not absolutes). Raw CSV: `{pre}_bench_launches.csv`.",
         f"Collected from `gpurun_out/{tag}` by `tools/collect_r2.py`.", "",
         "| launches | total ms | share | kernel |", "|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| {n} | {t:.3f} | {100 * t / tot:.1f} % | `{k[:110]}` |")

# ---- sweep kernel
sw = summary(os.path.join(src, "sweep_ws.ncu-rep"))
alg = bench["roofline"]["bytes_per_launch"]
peak = bench["roofline"]["peak"]
lines += ["", "## Sweep kernel (`sweep_ws`), full capture", "",
          f"`ncu --set full` of one 1,024-set ftp sweep (`tools/sweep_probe.py 1024 1`): {sw['duration_ms']:.1f} ms "
          f"(serialised under ncu), DRAM {sw['dram_bytes'] / 1e9:.1f} GB per launch against {alg / 1e9:.1f} GB algorithmic "
          f"({sw['dram_bytes'] / alg:.2f}x), {sw['dram_bytes'] / sw['duration_ms'] / 1e6:.0f} GB/s = "
          f"{100 * sw['dram_bytes'] / sw['duration_ms'] / 1e6 / peak:.0f} % of the measured {peak:.0f} GB/s copy bandwidth; "
          f"ncu DRAM throughput {sw['dram_pct']:.1f} % of its own peak; {sw['regs']:.0f} registers.",
          f"Stall mix: {sw['stalls']}.",
          f"The bench line's own CUDA-event timing of the kernel: {bench['roofline']['kernel_ms']:.1f} ms, "
          f"{bench['roofline']['achieved']:.0f} GB/s algorithmic, frac {bench['roofline']['frac']:.3f}."]
json.dump({"kernel": "sweep_ws", "sets": 1024, "dram_bytes_per_launch": sw["dram_bytes"],
           "source": f"ncu --set full of sweep_ws<1,1,double> with 1,024 ftp sets (tools/sweep_probe.py 1024 1, "
                     f"gpurun_out/{tag}): dram__bytes_read.sum + dram__bytes_write.sum in {sw['duration_ms']:.1f} ms"},
          open(os.path.join(prof, "traffic.json"), "w"))

# ---- single-graph kernels (entries of configs without a capture here are kept)
try:
    l2 = json.load(open(os.path.join(prof, "l2_traffic.json")))
except (OSError, ValueError):
    l2 = {}
lines += ["", "## Single-graph kernels, full captures", "",
          "`ncu --set full --launch-skip 3 --launch-count 1 -k 'regex:pslot|parall|persistent' python tools/time_probe.py <config> 2` "
          "(one launch = one whole run to convergence).", "",
          "| config | kernel | ms (ncu) | L2 sectors x 32 B | L1 ld / st sectors | DRAM bytes | warp instr | issue active | regs | stall mix |",
          "|---|---|---|---|---|---|---|---|---|---|"]
for c in ("C4-PARALL", "C1", "C4-SEQFIX", "C2", "C3"):
    rep = os.path.join(src, f"ncu_{c}.ncu-rep")
    if not os.path.exists(rep):
        continue
    s = summary(rep)
    kname = s["kernel"].replace("(KParams)", "").replace("void ", "").replace("hbp::", "") or "?"
    l2b = s["l2_sectors"] * 32
    l2[c] = {"l2_bytes_per_launch": l2b, "kernel": kname,
             "source": f"ncu --set full lts__t_sectors.sum x 32 B of one launch ({pre}, gpurun_out/{tag})"}
    lines.append(f"| {c} | `{kname}` | {s['duration_ms']:.3f} | {l2b / 1e9:.3f} GB | {s['l1_ld_sectors'] / 1e6:.1f} M / "
                 f"{s['l1_st_sectors'] / 1e6:.1f} M | {s['dram_bytes'] / 1e6:.1f} MB | {s['inst'] / 1e6:.1f} M | "
                 f"{s['issue_active_pct']:.1f} % | {s['regs']:.0f} | {s['stalls']} |")
lines += ["", "C1's row is the counter-barrier path: `lbp_pslot` runs C1 as one 8-CTA thread-block cluster "
          "with the hardware cluster barrier (`tools/time_probe.py`: 0.352 ms), but ncu's kernel replay launches "
          "it without the cluster attribute, and the kernel then takes the global-memory counter barrier (it "
          "checks `%cluster_nctarank` against the grid)."]
json.dump(l2, open(os.path.join(prof, "l2_traffic.json"), "w"), indent=1)
open(os.path.join(prof, f"{pre}_bench_launches.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
