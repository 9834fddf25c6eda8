"""Summarise an ncu report: key metrics + top SASS stall sites with source lines."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "Elapsed Cycles", "SM Frequency", "Executed Instructions", "Executed Ipc Active",
        "L2 Cache Throughput", "DRAM Throughput", "Registers Per Thread", "Achieved Occupancy",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate", "Branch Efficiency",
        "Avg. Divergent Branches", "Avg. Active Threads Per Warp"]
for row in csv.reader(io.StringIO(det)):
    if len(row) > 3 and row[-4] in want:
        print(f"  {row[-4]}: {row[-2]} {row[-3]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = None
for i, r in enumerate(rows):
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r; start = i + 1; break
if hdr is None:
    print("no source page"); sys.exit()
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
data = [r for r in rows[start:] if len(r) == len(hdr)]
tot = sum(int(r[i_s]) if r[i_s].strip("-").isdigit() else 0 for r in data)
print("  total stall samples", tot)
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.Counter()
for r in data:
    for c in stall_cols:
        v = r[hdr.index(c)]
        if v and v.isdigit():
            agg[c] += int(v)
print("  stalls:", ", ".join(f"{k[6:]}={100*v/max(1,tot):.1f}%" for k, v in agg.most_common(8)))
top = sorted(data, key=lambda r: -(int(r[i_s]) if r[i_s].isdigit() else 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    n = int(r[i_s]) if r[i_s].isdigit() else 0; print(f"  {n:7d} {100*n/max(1,tot):5.1f}%  {r[i_src].strip()[:110]}")
