"""Per-source-line instruction / stall breakdown of an ncu report (cuda,sass view)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None; fname = None; out = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            out.append((fname, int(r[0]), r[1][:95], int(d["Warp Stall Sampling (All Samples)"] or 0),
                        int(d["Instructions Executed"] or 0)))
        except ValueError:
            pass
ts = sum(o[3] for o in out) or 1; ti = sum(o[4] for o in out) or 1
print(f"instructions {ti/1e6:.1f} M, stall samples {ts}")
for o in sorted(out, key=lambda o: -o[4])[:n]:
    print(f"{o[0][:10]:10s} {o[1]:5d} inst {100*o[4]/ti:5.1f}% stall {100*o[3]/ts:5.1f}%  {o[2]}")
