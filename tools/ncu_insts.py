"""Per CUDA source line: warp instructions executed (ncu --page source).  Shows where a
kernel's instruction budget goes.  Usage: python tools/ncu_insts.py REPORT [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(k for k, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iI = hdr.index("Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[hi + 1:]:
    if len(r) > iI and r[iI].replace(".", "").isdigit():
        lines.append((float(r[iI]), int(r[iS]) if r[iS].isdigit() else 0, r[0], r[1]))
tot = sum(x[0] for x in lines)
print(f"total warp instructions {tot:.0f}")
for ins, smp, ln, src in sorted(lines, key=lambda x: -x[0])[:n]:
    print(f"{ins:12.0f} {100 * ins / tot:5.1f}%  samples {smp:6d}  L{ln:<5s} {src.strip()[:90]}")
