"""Aggregate ncu source-page metrics per CUDA source line (sass,cuda view)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
out = []
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[2] != "-":
        continue  # keep only source-line aggregate rows
    ie = int(r[7] or 0) if r[7].isdigit() else 0
    s = int(r[4]) if r[4].isdigit() else 0
    out.append((ie, s, r[0], r[1].strip()[:90]))
tot = sum(o[0] for o in out)
stot = sum(o[1] for o in out)
print("total executed warp instructions:", tot, "samples:", stot)
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "samples" else 0
for ie, s, l, t in sorted(out, key=lambda o: -o[key])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{ie:11d} {100*ie/max(1,tot):5.1f}%  samp {100*s/max(1,stot):5.1f}%  L{l:>4}  {t}")
