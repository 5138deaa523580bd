"""Fig. 7 / Table 3 analogs: summarise tools/big_check.py outputs (one B200) next to the
paper's K40c numbers.  Usage: python tools/paper_graphs_table.py FILE..."""
import re
import sys
PAPER = {"C2_ef64": ("rmat_s22_e64", 101038, 4.781), "S23E32": ("rmat_s23_e32", 58417, 8.655),
         "S24E16": ("rmat_s24_e16", 31327, 16.59), "K21": ("kron_g500-logn21", 44550, 4.088),
         "RGG24": ("rgg_n_24", 92.59, 2991.0), "C2": ("(not in the paper)", None, None)}
print("| graph (ours) | paper graph | n | nnz | sources | mean ms / BFS | GTEPS (nnz/time) | oracle check | paper K40c GTEPS (ms) |")
print("|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    t = open(f).read()
    m = re.search(r"^(\S+): n=(\d+) nnz=(\d+)", t, re.M)
    cfg, n, nnz = m.group(1), int(m.group(2)), int(m.group(3))
    mm = re.search(r"mean ([\d.]+) us -> ([\d.]+) GTEPS", t)
    ns = len(re.findall(r"^src \d+: [\d.]+ us, [\d.]+ GTEPS", t, re.M))
    ok = "bit-exact + Graph500-valid" if "graph500 validation of parents: ok" in t else "FAILED/absent"
    pg, mteps, pms = PAPER.get(cfg, ("?", None, None))
    paper = f"{mteps/1000:.3g} ({pms} ms)" if mteps else "-"
    print(f"| {cfg} | {pg} | {n:,} | {nnz:,} | {ns} | {float(mm.group(1))/1000:.3f} | {float(mm.group(2)):.1f} | {ok} | {paper} |")
