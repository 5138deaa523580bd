"""Aggregate ncu warp-stall samples per CUDA source line (ncu --page source cuda,sass)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr_i = next(k for k, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
iS = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[hdr_i + 1:]:
    if len(r) > iS and r[0] not in ("", "Line No") and r[iS].isdigit():
        lines.append((int(r[iS]), int(r[0]), r[1]))
tot = sum(x[0] for x in lines)
print("total samples", tot)
for s, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{s:7d} {100*s/tot:5.1f}%  L{ln:<5d} {src.strip()[:110]}")
