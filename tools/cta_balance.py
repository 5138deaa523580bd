"""Per-level, per-CTA phase durations of a BFS (load-balance / fixed-cost diagnostic).
For each level: the level's barrier-to-barrier time (CTA 0), the CTAs' work-phase times
(loop top to the counter flush; min / median / max), and the remainder = level time - max
work = counter flush + grid barrier + counter read + decision (the per-level fixed cost).
Usage: python tools/cta_balance.py [CONFIG] [NSOURCES] [norelabel] [noflush]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_1804_03327_b200 as pp

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = synth.make(cfg)
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g, relabel="norelabel" not in sys.argv)
depth = torch.empty(g.n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
LV = 64
pp.pp_bfs_debug_times(G.handle, LV)
for s in synth.sources(g, nsrc, seed=2):
    s = int(s)
    for _ in range(2):
        pp.bfs(G, s, depth)
    if "noflush" not in sys.argv:
        flush.zero_()
    torch.cuda.synchronize()
    st = pp.bfs(G, s, depth, stats_capacity=LV)
    t = pp.pp_bfs_debug_times(G.handle, LV, fetch=True)
    ph = pp.pp_bfs_debug_phases(G.handle, LV, t.shape[1])
    print(f"{cfg} source {s}: init {st['init_ns']/1e3:.1f} us; per level: barrier-to-barrier time (CTA 0), "
          f"warp-0 work max, CTA-wide work (all warps) p50/max, barrier release seen p50/max")
    for k in range(min(st["levels"], LV)):
        row = t[k] / 1e3
        cw, br = ph[1][k] / 1e3, ph[2][k] / 1e3
        lv = st["ns"][k] / 1e3
        print(f"  L{k+1} {'HL'[st['dir'][k]]} c={st['c'][k]:>8} level {lv:6.1f} | warp0 {row.max():5.1f} | "
              f"CTA {np.median(cw):5.1f}/{cw.max():5.1f} | released {np.median(br):5.1f}/{br.max():5.1f}")
