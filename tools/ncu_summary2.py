"""Summarise an lbp_persistent ncu report: key metrics, stall mix, SASS opcode mix.
Usage: python tools/ncu_summary2.py <report.ncu-rep>"""
import collections, csv, io, re, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "lts__t_sectors.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
for i, n in enumerate(h):
    if n in want:
        print(f"{n:60s} {v[i]}")
stalls = {n: v[i] for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
tot = sum(float(x or 0) for x in stalls.values())
top = sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:10]
print("stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={100*float(x)/tot:.1f}%" for k, x in top))
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
ii = hdr.index("Instructions Executed"); si = hdr.index("Source")
byop = collections.Counter(); totn = 0
for r in rows[2:]:
    if len(r) <= ii:
        continue
    try:
        n = int(r[ii])
    except ValueError:
        continue
    op = re.sub(r'^@!?U?P\w+\s+', '', r[si].strip())
    base = op.split()[0].split('.')[0] if op else '?'
    byop[base] += n
    totn += n
print("opcodes:", ", ".join(f"{k} {100*x/totn:.1f}%" for k, x in byop.most_common(16)))
