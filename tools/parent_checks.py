"""SURVEY pin P8 / P:266: "it took on average 79 parent checks before a valid parent was found
... after 2 BFS iterations, the average number of parents examined before a valid parent was
found dropped from 79 to 1.3".  Counted from the definition on the CPU (oracle depths; rows in
the caller's sorted order, as the paper's row-based pull scans them): in a pull-only BFS, level
k examines, for every vertex it discovers, its in-neighbours in order up to the first one at
depth <= k; the count is that first-hit position (1-based).  Printed per level: discovered
vertices, mean parent checks among them, and (the GPU's layout) the same under the
PP_GRAPH_RELABEL degree order.  Usage: python tools/parent_checks.py [CONFIG] [SOURCES]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "K21"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = synth.make(cfg)
n = g.n
deg = np.diff(g.off)
rows = np.repeat(np.arange(n), deg)
pos = np.arange(g.nnz) - g.off[rows]
key = synth.degree_order_key(g).astype(np.int64)
# relabelled order: position of each entry within its row after sorting the row by key
order = np.lexsort((key[g.idx], rows))
rpos = np.empty(g.nnz, np.int64)
rpos[order] = np.arange(g.nnz) - g.off[rows[order]]
print(f"{cfg}: n={n} nnz={g.nnz}; pull-only BFS, parent checks per discovered vertex (1-based "
      f"position of the first in-neighbour already visited)")
print("| source | level | discovered | mean checks (caller order) | mean checks (degree order) |")
print("|---|---|---|---|---|")
for s in synth.sources(g, S, seed=2):
    d, L = oracle.bfs(g, int(s))
    dj = d[g.idx]
    for k in range(1, L):
        found = d == k + 1
        hit = (dj >= 1) & (dj <= k) & found[rows]
        first = np.full(n, np.iinfo(np.int64).max)
        np.minimum.at(first, rows[hit], pos[hit])
        rfirst = np.full(n, np.iinfo(np.int64).max)
        np.minimum.at(rfirst, rows[hit], rpos[hit])
        c = int(found.sum())
        if c == 0:
            continue
        print(f"| {s} | {k} | {c} | {(first[found] + 1).mean():.2f} | {(rfirst[found] + 1).mean():.2f} |")
