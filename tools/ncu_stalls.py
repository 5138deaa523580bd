"""Per CUDA source line: warp-stall samples split by reason (ncu --page source cuda,sass).
Usage: python tools/ncu_stalls.py REPORT.ncu-rep [N]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(k for k, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [(k, h) for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot_r = collections.Counter()
lines = []
for r in rows[hi + 1:]:
    if len(r) > iS and r[0] not in ("", "Line No") and r[iS].isdigit():
        c = {h[6:]: int(r[k]) for k, h in reasons if r[k].isdigit() and int(r[k])}
        tot_r.update(c)
        lines.append((int(r[iS]), int(r[0]), r[1], c))
tot = sum(x[0] for x in lines)
print("total samples", tot, " by reason:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in tot_r.most_common(10)))
for s, ln, src, c in sorted(lines, key=lambda x: -x[0])[:n]:
    top = ", ".join(f"{k} {v}" for k, v in sorted(c.items(), key=lambda x: -x[1])[:3])
    print(f"{s:7d} {100*s/tot:5.1f}%  L{ln:<5d} {src.strip()[:80]:80s} [{top}]")
