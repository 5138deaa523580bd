"""Per-level, per-CTA phase durations of one BFS (load-balance diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

src = int(sys.argv[1]) if len(sys.argv) > 1 else 2764614
g = synth.make(sys.argv[2] if len(sys.argv) > 2 else "C2")
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g)
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
LV = 16
pp.pp_bfs_debug_times(G.handle, LV)
for _ in range(3):
    st = pp.bfs(G, src, depth, stats_capacity=64)
t = pp.pp_bfs_debug_times(G.handle, LV, fetch=True)
for k in range(st["levels"]):
    row = t[k] / 1e3
    print(f"L{k+1} {'HL'[st['dir'][k]]} level {st['ns'][k]/1e3:7.1f} us | CTA work min {row.min():6.1f} "
          f"p50 {np.median(row):6.1f} p90 {np.percentile(row,90):6.1f} max {row.max():6.1f} (cta {row.argmax()})")
