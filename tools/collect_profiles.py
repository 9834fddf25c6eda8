"""Copy one gpu_round.sh output (gpurun_out/<tag>) into profiles/: the bench
line and the reference arm, the launch list (CSV + per-kernel summary), the
sweep kernel's full-capture summary and its DRAM traffic (profiles/traffic.json,
read by bench.py). Usage: python tools/collect_profiles.py <tag>"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out", tag)
prof = os.path.join(ROOT, "profiles")

bench = json.load(open(os.path.join(src, "bench.json")))
json.dump(bench, open(os.path.join(prof, "r1_bench_n1.json"), "w"), indent=1)
ref = json.load(open(os.path.join(src, "bench_ref.json")))
json.dump(ref, open(os.path.join(prof, "r1_bench_ref_n1.json"), "w"), indent=1)

# launch list
raw = open(os.path.join(src, "launches.csv")).read()
open(os.path.join(prof, "r1_bench_launches.csv"), "w").write(raw)
rows = [r for r in csv.reader(io.StringIO(raw)) if len(r) > 5][1:]
agg = collections.OrderedDict()
for r in rows:
    a = agg.setdefault(r[4], [0, 0.0])
    a[0] += 1
    a[1] += float(r[-1]) / 1e6
tot = sum(a[1] for a in agg.values())
lines = ["# r1 — launch list of `python bench.py --steps 2 --warmup 3` (first 120 launches)", "",
         "`ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv python bench.py --steps 2 --warmup 3`",
         "(cold-cache, serialised per-launch times: compare shares, not absolutes). Raw CSV: `r1_bench_launches.csv`.",
         f"Collected from `gpurun_out/{tag}` by `tools/collect_profiles.py`.", "",
         "| launches | total ms | share | kernel |", "|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| {n} | {t:.3f} | {100 * t / tot:.1f} % | `{k[:100]}` |")

# sweep kernel full capture
rep = os.path.join(src, "sweep_ws.ncu-rep")
raw_csv = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
r = list(csv.reader(io.StringIO(raw_csv)))
h, v = r[0], r[2]
get = lambda k: float(v[h.index(k)].replace(",", ""))
rd = get("dram__bytes_read.sum")
wr = get("dram__bytes_write.sum")
unit = r[1][h.index("dram__bytes_read.sum")]
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Tbyte": 1e12, "byte": 1.0}[unit]
dur_ms = get("gpu__time_duration.sum") / (1e6 if r[1][h.index("gpu__time_duration.sum")] == "ns" else 1.0)
traffic = (rd + wr) * scale
alg = bench["roofline"]["bytes_per_launch"]
peak = bench["roofline"]["peak"]
lines += ["",
          "The sweep kernel dominates device time: one launch per sweep of 1,024 sets.",
          f"Full capture (`ncu --set full`, 1,024 sets, `tools/sweep_probe.py 1024 1`): {dur_ms:.1f} ms, "
          f"DRAM {rd * scale / 1e9:.1f} GB read + {wr * scale / 1e9:.1f} GB written = {traffic / 1e9:.1f} GB per launch "
          f"against {alg / 1e9:.1f} GB algorithmic ({traffic / alg:.2f}x), "
          f"{traffic / dur_ms / 1e6:.0f} GB/s = {100 * traffic / dur_ms / 1e6 / peak:.0f} % of the measured {peak:.0f} GB/s copy bandwidth.",
          f"The bench line's own CUDA-event timing of the same kernel: {bench['roofline']['kernel_ms']:.1f} ms, "
          f"{bench['roofline']['achieved']:.0f} GB/s algorithmic, frac {bench['roofline']['frac']:.3f}."]
open(os.path.join(prof, "r1_bench_launches.md"), "w").write("\n".join(lines) + "\n")
json.dump({"kernel": "sweep_ws", "sets": 1024, "dram_bytes_per_launch": traffic,
           "source": f"ncu --set full of sweep_ws<1,1,double> with 1,024 ftp sets (tools/sweep_probe.py 1024 1, "
                     f"gpurun_out/{tag}): dram__bytes_read.sum + dram__bytes_write.sum in {dur_ms:.1f} ms"},
          open(os.path.join(prof, "traffic.json"), "w"))
print("\n".join(lines))
